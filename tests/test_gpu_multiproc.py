"""GPU, two PROCESSES on cuda:0: the cross-process path of the document-sharded store.

Process A owns the chunks: it ingests them into its HBM store and exports its directory blob
(tkv_store_export_directory: ids, page lists, framed tokens, its pool's CUDA-IPC handle, fingerprint, geometry).
Process B imports the blob (tkv_store_import_directory: cudaIpcOpenMemHandle of A's pool) and serves a request
whose chunks all live in A's store: the gather kernel reads them straight out of A's pool (on a multi-GPU box:
over NVLink). B's logits must equal, bit for bit, A's logits for the same request on its all-local store. B also
checks the validation: a blob from a different model is StaleCacheError, a corrupted page index FormatError.
"""
import multiprocessing as mp
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED, N_CHUNKS = 42, 6


def _payloads():
    import oracle as O
    return [O.random_text_tokens(9000 + i, n) for i, n in enumerate((126, 62, 200, 1, 90, 126))], \
        O.random_text_tokens(0xB10B, 24)


def _owner(dtype, q_out, q_in):
    from paper_2410_07590_b200 import turbokv as T
    eng = T.Engine(T.ModelConfig.toy(), SEED, dtype=dtype, store_capacity_tokens=4096)
    pays, query = _payloads()
    ids = eng.ingest_chunks(pays)
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        local = eng.prefill_query(ctx, query).copy()
    q_out.put({"blob": eng.export_directory(), "ids": ids, "logits": local})
    evict_err = None
    try:
        eng.store_evict(ids[0])  # shared with a peer now: must be refused
    except T.ConfigError as e:
        evict_err = str(e)
    q_out.put({"evict_refused": evict_err is not None})
    q_in.get(timeout=300)  # keep the pool alive until the peer is done
    eng.close()


def _peer(dtype, blob, ids, q_out):
    from paper_2410_07590_b200 import turbokv as T
    pays, query = _payloads()
    res = {}
    eng = T.Engine(T.ModelConfig.toy(), SEED, dtype=dtype, store_capacity_tokens=4096)
    eng.import_directory(1, blob)
    res["all_remote"] = all(eng.store_contains(i) for i in ids) and eng.store_count()[1] == 0
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        res["logits"] = eng.prefill_query(ctx, query).copy()
    res["remote_bytes"] = eng.remote_bytes()
    # naive path over the peer's token records (framed tokens travel in the blob)
    res["naive_ok"] = np.isfinite(eng.naive_prefill_ids(ids, query, T.MaskMode.Causal).last_logits).all()
    # validation: another model's directory, a page index outside the pool
    other = T.Engine(T.ModelConfig.toy(), SEED + 1, dtype=dtype, store_capacity_tokens=512)
    try:
        other.import_directory(1, blob)
        res["stale"] = None
    except T.StaleCacheError:
        res["stale"] = "StaleCacheError"
    other.close()
    bad = bytearray(blob)
    head = struct.calcsize("<4sIQQqq64sq")
    struct.pack_into("<i", bad, head + 24, 10 ** 9)  # first entry's first page index
    eng2 = T.Engine(T.ModelConfig.toy(), SEED, dtype=dtype, store_capacity_tokens=512)
    try:
        eng2.import_directory(1, bytes(bad))
        res["corrupt"] = None
    except T.FormatError:
        res["corrupt"] = "FormatError"
    res["nothing_registered"] = eng2.store_contains(ids[0]) is False
    eng2.close()
    eng.close()
    q_out.put(res)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_two_process_ipc_store_bitwise(dtype):
    ctx = mp.get_context("spawn")
    qa, qdone, qb = ctx.Queue(), ctx.Queue(), ctx.Queue()
    a = ctx.Process(target=_owner, args=(dtype, qa, qdone))
    a.start()
    try:
        first = qa.get(timeout=300)
        b = ctx.Process(target=_peer, args=(dtype, first["blob"], first["ids"], qb))
        b.start()
        res = qb.get(timeout=300)
        b.join(timeout=60)
        second = qa.get(timeout=60)
    finally:
        qdone.put(1)
        a.join(timeout=60)
    assert res["all_remote"]
    assert np.array_equal(res["logits"], first["logits"])  # peer-pool gather == local gather, bit for bit
    assert res["remote_bytes"] > 0 and res["naive_ok"]
    assert res["stale"] == "StaleCacheError" and res["corrupt"] == "FormatError" and res["nothing_registered"]
    assert second["evict_refused"]
