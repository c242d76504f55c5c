"""Generate the LARGE golden fixtures (tests/golden/golden_large.{json,npz}) with the UNMODIFIED reference.

These pin the CUDA path at the regimes the headline configs run in (VERDICT r1 "next round" #1), where the
small goldens of make_golden.py do not reach:

  * ``c2ctx``  — BASELINE configs[1]'s context regime at exact Qwen2-7B dims with 2 layers: 16 chunks x 512
    framed tokens (P = 8192 cached tokens) + a 64-token query, reordered AND composite positions. Besides
    the first-token logits it records sampled rows of the reference's ROTATED keys / values of both layers
    (rows spread over all 8192 positions) and 4 greedy-decode tokens.
  * ``llama1`` — Llama-3-8B dims (H32 / Hkv8, d 128, hidden 4096, inter 14336, rope base 5e5), 1 layer,
    6 chunks x 64 framed tokens (the C4 chunk shape) + a 16-token query, all four paths.
  * ``c3b``    — BASELINE configs[2]'s shape at exact Qwen2-7B dims with 1 layer: a 24-chunk corpus of
    800-token framed chunks, 4 requests that each retrieve 20 of them (different subsets and orders) with
    their own 64-token query, composite and reordered (the batched prefill path).

The reference is single-threaded f64 (~1.2 GFLOP/s), so chunk ingest is spread over worker PROCESSES that
share one TKVC store directory (content-addressed, atomic writes: proj/src/kvstore.cpp:78-132); the final
assemble + prefill_query of every request runs in workers too. ~30 min on 8 cores. Run here (where
/root/reference exists):  python tests/golden/make_golden_large.py [--workers 7]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor
import multiprocessing as mp

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

LLAMA1 = O.Cfg(1, 32, 8, 128, 4096, 14336, 259, 500000.0, 1e-5)


def case_defs():
    q2 = O.qwen_layers(2)
    q1 = O.qwen_layers(1)
    c2 = {
        "cfg": q2, "seed": 42,
        "payloads": [O.random_text_tokens(5000 + i, 510) for i in range(16)],
        "requests": [{"chunks": list(range(16)), "query": O.random_text_tokens(0xC2C2, 64)}],
        "naive": False, "kv_rows": True, "decode": 4,
    }
    ll = {
        "cfg": LLAMA1, "seed": 7,
        "payloads": [O.random_text_tokens(6000 + i, 62) for i in range(6)],
        "requests": [{"chunks": list(range(6)), "query": O.random_text_tokens(0x11A3A, 16)}],
        "naive": True, "kv_rows": True, "decode": 4,
    }
    rng = np.random.default_rng(0xC3)
    reqs = []
    for r in range(4):
        sel = rng.permutation(24)[:20].tolist()
        reqs.append({"chunks": sel, "query": O.random_text_tokens(0xC300 + r, 64)})
    c3 = {
        "cfg": q1, "seed": 42,
        "payloads": [O.random_text_tokens(7000 + i, 798) for i in range(24)],
        "requests": reqs, "naive": False, "kv_rows": False, "decode": 0,
    }
    return {"c2ctx": c2, "llama1": ll, "c3b": c3}


_ENG = {}


def _engine(name, store):
    if name not in _ENG:
        for k in list(_ENG):
            _ENG.pop(k).close()
        c = case_defs()[name]
        _ENG[name] = O.RefEngine(c["cfg"], c["seed"], store)
    return _ENG[name]


def ingest_task(args):
    name, store, i = args
    t = time.time()
    eng = _engine(name, store)
    cid = eng.ingest(case_defs()[name]["payloads"][i])
    return name, i, cid, time.time() - t


def kv_sample_rows(P: int, n: int = 64) -> np.ndarray:
    """Rows spread over every chunk of the context: chunk starts/ends and interior points."""
    return np.unique(np.linspace(0, P - 1, n).astype(np.int64))


def request_task(args):
    name, store, r, reordered, ids = args
    t = time.time()
    c = case_defs()[name]
    eng = _engine(name, store)
    out, arrays = {}, {}
    tag = "reordered" if reordered else "composite"
    key = f"{name}.r{r}.{tag}"
    ctx = eng.assemble(ids, reordered)
    pos, nxt = ctx.positions()
    arrays[f"{key}.positions"] = pos
    out[f"r{r}.{tag}.next_position"] = nxt
    if c["kv_rows"] and reordered:
        rows = kv_sample_rows(len(pos))
        arrays[f"{name}.kv_rows"] = rows
        for layer in range(c["cfg"].layer_num):
            arrays[f"{name}.krot{layer}"] = ctx.kv(layer, 2)[rows]
            arrays[f"{name}.v{layer}"] = ctx.kv(layer, 1)[rows]
    logits, flops = ctx.prefill_query(c["requests"][r]["query"])
    arrays[f"{key}.logits"] = logits
    out[f"r{r}.{tag}.flops"] = [int(x) for x in flops]
    if c["decode"] and reordered:
        out[f"r{r}.decode"] = [int(t) for t in ctx.greedy_decode(c["decode"])]
    ctx.close()
    return name, out, arrays, time.time() - t


def naive_task(args):
    name, store, r, independent = args
    t = time.time()
    c = case_defs()[name]
    eng = _engine(name, store)
    framed = [O.frame(c["payloads"][i]) for i in c["requests"][r]["chunks"]]
    tag = "independent" if independent else "causal"
    logits = eng.naive_prefill(framed, c["requests"][r]["query"], independent)
    return name, {}, {f"{name}.r{r}.naive_{tag}.logits": logits}, time.time() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=7)
    ap.add_argument("--cases", default="c2ctx,llama1,c3b")
    args = ap.parse_args()
    O.build(ref=True)
    defs = case_defs()
    names = args.cases.split(",")
    stores = {n: tempfile.mkdtemp(prefix=f"tkv-golden-{n}-") for n in names}
    ctx = mp.get_context("spawn")
    meta: dict = {}
    arrays: dict = {}
    with ProcessPoolExecutor(args.workers, mp_context=ctx) as ex:
        tasks = [(n, stores[n], i) for n in names for i in range(len(defs[n]["payloads"]))]
        ids = {n: [None] * len(defs[n]["payloads"]) for n in names}
        for n, i, cid, dt in ex.map(ingest_task, tasks):
            ids[n][i] = cid
            print(f"ingest {n}[{i}] {dt:.0f}s", flush=True)
        jobs = []
        for n in names:
            c = defs[n]
            meta[n] = {"seed": c["seed"], "config": c["cfg"].__dict__, "ids": [f"{x:016x}" for x in ids[n]],
                       "requests": [{"chunks": q["chunks"]} for q in c["requests"]]}
            arrays[f"{n}.payloads"] = np.concatenate(c["payloads"]).astype(np.int32)
            arrays[f"{n}.payload_offsets"] = np.concatenate(
                [[0], np.cumsum([len(p) for p in c["payloads"]])]).astype(np.int64)
            for r, q in enumerate(c["requests"]):
                arrays[f"{n}.r{r}.query"] = np.asarray(q["query"], np.int32)
                rid = [ids[n][i] for i in q["chunks"]]
                for reordered in (True, False):
                    jobs.append(ex.submit(request_task, (n, stores[n], r, reordered, rid)))
                if c["naive"]:
                    for independent in (False, True):
                        jobs.append(ex.submit(naive_task, (n, stores[n], r, independent)))
        for j in jobs:
            n, out, arr, dt = j.result()
            meta[n].update(out)
            arrays.update(arr)
            print(f"request {n} {sorted(arr)[0]} {dt:.0f}s", flush=True)
    for n in names:
        meta[n]["fingerprint"] = f"{O.Ref.identity(defs[n]['cfg'], defs[n]['seed'])[1]:016x}"
    npz = os.path.join(HERE, "golden_large.npz")
    js = os.path.join(HERE, "golden_large.json")
    if os.path.exists(js):  # merge with cases generated by an earlier partial run
        old = json.load(open(js))
        old.update(meta)
        meta = old
        with np.load(npz) as z:
            prev = {k: z[k] for k in z.files if k.split(".")[0] not in names}
        prev.update(arrays)
        arrays = prev
    np.savez_compressed(npz, **arrays)
    with open(js, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays;", os.path.getsize(npz), "bytes")


if __name__ == "__main__":
    main()
