"""CPU, world_size 2 over gloo: the multi-GPU host logic (paper_2410_07590_b200/sharding.py) — document
ownership, directory-blob exchange (the tkv_store_export_directory layout), remote registration under peer slots, locality routing.
The engine is a stand-in with the Engine method surface (no GPU here); the GPU side of remote chunks
(gather kernel reading a peer pool) is covered by tests/test_gpu_parity.py::test_remote_chunks_*."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_07590_b200 import sharding as S
from paper_2410_07590_b200 import turbokv as T

FP = 0x8DD32810BD252FD1  # toy seed-42 model fingerprint


class FakeEngine:
    def __init__(self, rank):
        self.rank, self.pages, self.attached, self.remote, self.fetched = rank, {}, {}, {}, []

    def fingerprint(self):
        return FP

    def ingest_chunks(self, payloads):
        ids = []
        for p in payloads:
            cid = T.chunk_content_id(T.frame_chunk(p), FP)
            self.pages[cid] = (np.arange((len(p) + 2 + 63) // 64, dtype=np.int32) + 100 * self.rank, len(p) + 2)
            ids.append(cid)
        return ids

    def chunk_pages(self, cid):
        return self.pages[cid]

    def export_directory(self):  # the engine's blob layout (include/tkv.h), built host-side
        return S.pack_directory(FP, 64 * 1024, 64, 1000, bytes([self.rank]) * 64,
                                [(c, n, p, None) for c, (p, n) in self.pages.items()])

    def import_directory(self, slot, blob):  # what tkv_store_import_directory validates and registers
        d = S.parse_directory(blob)
        assert d["fingerprint"] == FP and d["page_tokens"] == 64
        self.attached[slot] = d["ipc"]
        for cid, length, pages, framed in d["entries"]:
            assert all(0 <= p < d["pool_pages"] for p in pages)
            self.remote[cid] = (slot, length, list(pages), framed)

    def fetch_remote(self, cid):
        self.fetched.append(cid)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    payloads = [rng.integers(97, 123, int(n)).astype(np.int32) for n in (10, 200, 63, 64, 5, 130)]
    docs = [f"doc-{i // 2}" for i in range(6)]  # two chunks per document
    eng = FakeEngine(rank)
    st = S.ShardedStore(eng, rank, world)
    ids = st.ingest(payloads, docs)
    st.exchange()
    owners = {cid: S.owner_of(d, world) for cid, d in zip(ids, docs)}
    out = {
        "all_known": sorted(st.directory) == sorted(ids),
        "owners_ok": all(st.directory[c].owner == owners[c] for c in ids),
        "remote_ok": sorted(eng.remote) == sorted(c for c in ids if owners[c] != rank),
        "slots": sorted({v[0] for v in eng.remote.values()}),
        "attached": {k: v[0] for k, v in eng.attached.items()},
        "pages_ok": all(list(eng.remote[c][2]) == list(st.directory[c].pages) for c in eng.remote),
        "route": st.route(ids[:2]),
        "route_owner": owners[ids[1]],  # the 200-token chunk dominates the first request
        "docs_colocated": all(owners[ids[2 * i]] == owners[ids[2 * i + 1]] for i in range(3)),
    }
    st.cache_remote(ids)
    out["fetched"] = sorted(eng.fetched) == sorted(c for c in ids if owners[c] != rank)
    out["after_cache_remote"] = st.remote_fraction(ids)
    q.put((rank, out))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_directory_exchange_and_routing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank, out in results.items():
        assert out["all_known"] and out["owners_ok"] and out["remote_ok"] and out["pages_ok"], out
        assert out["docs_colocated"]
        assert out["slots"] in ([], [1]) and all(v == 1 - rank for v in out["attached"].values()), out
        assert out["route"] == out["route_owner"]
        assert out["fetched"] and out["after_cache_remote"] == 0.0


def test_owner_is_deterministic_and_balanced():
    counts = np.bincount([S.owner_of(f"doc-{i}", 8) for i in range(4000)], minlength=8)
    assert counts.min() > 400 and S.owner_of("x", 1) == 0
    assert S.owner_of("doc-42", 8) == S.owner_of("doc-42", 8)
