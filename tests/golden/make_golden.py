"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The reference is compiled from its own sources into oracle/_ref by oracle/Makefile and
driven through oracle/ref_capi.cpp. /root/reference does not exist on the GPU box, so
the outputs are committed (golden.json + golden.npz) and the GPU tests read them.

Cases:
  * SplitMix64 canonical vectors (proj/docs/formats.md:45-52)
  * toy weight identity goldens (proj/tests/test_model.cpp:67-80, docs/formats.md:107-112)
  * assemble position ids for framed lengths 3,4,5 (proj/tests/test_pipeline.cpp:118-148)
  * masks: build_mask Causal/Independent and causal_rows (proj/src/attention.cpp:50-92)
  * C1 (BASELINE configs[0]): toy, 4 chunks x 128 framed + 32-token query, all four paths,
    plus assembled K/V (unrotated and rotated) of two layers
  * a ragged case in the style of proj/tests/acceptance_main.cpp:80-139 (1..64-token payloads)
  * exact Qwen2-7B dims with 1 layer (SURVEY §8c "parity at exact dims")
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def case_paths(name, cfg, seed, payloads, query, arrays, meta, kv_layers=()):
    d = tempfile.mkdtemp(prefix=f"tkv-golden-{name}-")
    eng = O.RefEngine(cfg, seed, d)
    ids = [eng.ingest(p) for p in payloads]
    framed = [O.frame(p) for p in payloads]
    out = {"ids": [f"{i:016x}" for i in ids], "fingerprint": f"{eng.fingerprint():016x}"}
    for reordered, tag in ((True, "reordered"), (False, "composite")):
        ctx = eng.assemble(ids, reordered)
        pos, nxt = ctx.positions()
        arrays[f"{name}.{tag}.positions"] = pos
        out[f"{tag}.next_position"] = nxt
        if reordered:
            for layer in kv_layers:
                arrays[f"{name}.k{layer}"] = ctx.kv(layer, 0)
                arrays[f"{name}.v{layer}"] = ctx.kv(layer, 1)
                arrays[f"{name}.krot{layer}"] = ctx.kv(layer, 2)
        logits, flops = ctx.prefill_query(query)
        arrays[f"{name}.turbo_{tag}.logits"] = logits
        out[f"turbo_{tag}.flops"] = [int(x) for x in flops]
        if reordered:
            out["decode8"] = [int(t) for t in ctx.greedy_decode(8)]
    for independent, tag in ((False, "causal"), (True, "independent")):
        arrays[f"{name}.naive_{tag}.logits"] = eng.naive_prefill(framed, query, independent)
    arrays[f"{name}.query"] = np.asarray(query, np.int32)
    arrays[f"{name}.payload_offsets"] = np.concatenate([[0], np.cumsum([len(p) for p in payloads])]).astype(np.int64)
    arrays[f"{name}.payloads"] = np.concatenate(payloads).astype(np.int32)
    out["seed"] = seed
    out["config"] = cfg.__dict__
    meta[name] = out
    eng.close()


def main():
    O.build(ref=True)
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {}

    meta["splitmix"] = {
        str(s): [f"{O.Ref.lib().ref_splitmix_at(s, i):016x}" for i in range(3)] for s in (0, 1234567, 42)
    }
    ck, fp, e00 = O.Ref.identity(O.TOY, 42)
    ck7, _, _ = O.Ref.identity(O.TOY, 7)
    meta["toy_identity"] = {"checksum42": f"{ck:016x}", "fingerprint42": f"{fp:016x}", "emb00": e00,
                            "checksum7": f"{ck7:016x}"}

    # positions pinned by proj/tests/test_pipeline.cpp:118-148 (payloads "a", "bc", "def")
    d = tempfile.mkdtemp(prefix="tkv-golden-pos-")
    eng = O.RefEngine(O.TOY, 42, d)
    ids = [eng.ingest([ord(c) for c in s]) for s in ("a", "bc", "def")]
    for reordered, tag in ((True, "reordered"), (False, "composite")):
        pos, nxt = eng.assemble(ids, reordered).positions()
        meta[f"positions_345.{tag}"] = {"positions": pos.tolist(), "next": nxt}
    eng.close()

    # masks as dense 0/1 from the reference itself
    for independent, tag in ((False, "causal"), (True, "independent")):
        arrays[f"mask.3452.{tag}"] = O.Ref.build_mask([3, 4, 5, 2], independent)
    arrays["mask.causal_rows_5_7"] = O.Ref.causal_rows(5, 7)

    # C1: toy, 4 x 126-byte payloads (128 framed) + 32-token query, seed 42
    c1_payloads = [O.random_text_tokens(1000 + i, 126) for i in range(4)]
    c1_query = O.random_text_tokens(0x51DEC0DE, 32)
    case_paths("c1", O.TOY, 42, c1_payloads, c1_query, arrays, meta, kv_layers=(0, 3))

    # ragged: 6 chunks with payload lengths 1..64 and a 17-token query, seed 99
    lens = [1, 64, 7, 33, 2, 50]
    rag = [O.random_text_tokens(2000 + i, n) for i, n in enumerate(lens)]
    case_paths("ragged", O.TOY, 99, rag, O.random_text_tokens(77, 17), arrays, meta, kv_layers=(1,))

    # exact Qwen2-7B dims, 1 layer: 3 chunks (30, 5, 61 payload) + 9-token query
    q1 = O.qwen_layers(1)
    qp = [O.random_text_tokens(3000 + i, n) for i, n in enumerate((30, 5, 61))]
    case_paths("qwen1", q1, 42, qp, O.random_text_tokens(88, 9), arrays, meta, kv_layers=(0,))

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays;", os.path.getsize(os.path.join(HERE, "golden.npz")), "bytes")


if __name__ == "__main__":
    main()
