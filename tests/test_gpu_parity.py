"""GPU parity: the CUDA path (libtkv_b200.so through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): layouts, position ids and masks bit-exact; fp32 logits and KV within
1e-4 relative; bf16 within 2e-2 with the first-token argmax identical whenever the oracle's top-1/top-2
margin exceeds the measured bf16 error (SURVEY §7 hard part 4).
"Relative" for fp32 is per element, |got-ref| <= 1e-4 * max(|ref|, 1e-2 * max|ref|) (a floor for
near-zero logits). For bf16 the floor is max|ref| itself, i.e. max|got-ref| <= 2e-2 * max|ref|:
bf16 carries 8 mantissa bits, so a per-element bound on logits near zero would test rounding noise.
"""
import os
import sys

import numpy as np
import pytest

import oracle as O
from paper_2410_07590_b200 import turbokv as T
from tests.tkvc_io import write_tkvc

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_TOL = 2e-2


def rel_excess(got, ref, floor_frac=1e-2):
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    scale = np.maximum(np.abs(ref), floor_frac * np.abs(ref).max())
    return float((np.abs(got - ref) / scale).max())


def assert_close(got, ref, tol):
    e = rel_excess(got, ref, floor_frac=1e-2 if tol <= FP32_TOL else 1.0)
    assert e <= tol, f"relative error {e:.3e} > {tol}"


def assert_argmax(got, ref, err_budget):
    ref = np.asarray(ref).ravel()
    got = np.asarray(got).ravel()
    top = np.sort(ref)[::-1]
    margin = (top[0] - top[1]) / np.abs(ref).max()
    if margin > err_budget:
        assert int(np.argmax(got)) == int(np.argmax(ref)), f"argmax differs with margin {margin:.3e}"


def cfg_t(meta) -> T.ModelConfig:
    return T.ModelConfig(**meta["config"])


def payloads(A, name):
    offs = A[f"{name}.payload_offsets"]
    return [A[f"{name}.payloads"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]


def to_bf16(x: np.ndarray) -> np.ndarray:
    """f64 -> f32 (RN) -> bf16 (RNE), returned as f32 — the engine's canonical cast."""
    f = np.asarray(x, np.float64).astype(np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


_ENGINES = {}


def engine(cfg: T.ModelConfig, seed: int, dtype: str, flags: int = 0) -> T.Engine:
    key = (tuple(vars(cfg).values()), seed, dtype, flags)
    if key not in _ENGINES:
        _ENGINES[key] = T.Engine(cfg, seed, dtype=dtype, flags=flags, store_capacity_tokens=1 << 16)
    return _ENGINES[key]


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("name", ["c1", "ragged"])
def test_four_paths_vs_golden(golden, name, dtype, tol):
    """C1 (BASELINE configs[0]) and a ragged grid: all four paths against the reference's logits."""
    meta, A = golden
    m = meta[name]
    eng = engine(cfg_t(m), m["seed"], dtype)
    assert f"{eng.fingerprint():016x}" == m["fingerprint"]
    ids = eng.ingest_chunks(payloads(A, name))
    assert [f"{i:016x}" for i in ids] == m["ids"]  # content ids bit-exact (kvstore.cpp:58-64)
    q = A[f"{name}.query"]
    for mode, tag in ((T.PositionMode.Reordered, "reordered"), (T.PositionMode.Composite, "composite")):
        with eng.assemble(ids, mode) as ctx:
            assert np.array_equal(ctx.positions, A[f"{name}.{tag}.positions"])
            assert ctx.next_position == m[f"{tag}.next_position"]
            logits = eng.prefill_query(ctx, q)[0]
            ref = A[f"{name}.turbo_{tag}.logits"]
            assert_close(logits, ref, tol)
            assert_argmax(logits, ref, tol)
    framed = [O.frame(p) for p in payloads(A, name)]
    for mode, tag in ((T.MaskMode.Causal, "causal"), (T.MaskMode.Independent, "independent")):
        logits = eng.naive_prefill(framed, q, mode, keep_context=False)[0]
        assert_close(logits, A[f"{name}.naive_{tag}.logits"], tol)


def test_turbo_equals_naive_independent_and_composite_defect(golden):
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], "f32")
    ids = eng.ingest_chunks(payloads(A, "c1"))
    q = A["c1.query"]
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        turbo = eng.prefill_query(ctx, q)[0]
    with eng.naive_prefill_ids(ids, q, T.MaskMode.Independent) as naive:
        oracle_logits = naive.last_logits[0]
    assert_close(turbo, oracle_logits, FP32_TOL)  # proj/tests/test_pipeline.cpp:182-208
    with eng.assemble(ids, T.PositionMode.Composite) as ctx:
        comp = eng.prefill_query(ctx, q)[0]
    assert np.abs(comp - oracle_logits).max() > 1e-3  # composite defect, test_pipeline.cpp:210-234


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_empty_context_equals_vanilla_prefill(golden, dtype):
    """Assembling zero chunks and prefilling the query is bitwise the vanilla prefill of the query alone
    (proj/tests/test_pipeline.cpp:165-180)."""
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], dtype)
    q = A["c1.query"]
    with eng.assemble([], T.PositionMode.Reordered) as ctx:
        assert ctx.total_tokens() == 0 and ctx.next_position == 0
        turbo = eng.prefill_query(ctx, q)[0]
    vanilla = eng.naive_prefill([], q, T.MaskMode.Causal, keep_context=False)[0]
    assert np.array_equal(turbo, vanilla)


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_single_chunk_four_paths_agree(golden, dtype, tol):
    """With one retrieved chunk composite == reordered positions and the causal mask == the independent one, so
    all four paths give the same logits (proj/tests/acceptance_main.cpp:447-471)."""
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], dtype)
    pay = payloads(A, "c1")[:1]
    ids = eng.ingest_chunks(pay)
    q = A["c1.query"]
    outs = []
    for mode in (T.PositionMode.Reordered, T.PositionMode.Composite):
        with eng.assemble(ids, mode) as ctx:
            outs.append(eng.prefill_query(ctx, q)[0])
    for mask in (T.MaskMode.Causal, T.MaskMode.Independent):
        outs.append(eng.naive_prefill([O.frame(p) for p in pay], q, mask, keep_context=False)[0])
    assert np.array_equal(outs[0], outs[1])  # identical positions -> identical gather and prefill
    assert np.array_equal(outs[2], outs[3])  # identical masks
    assert_close(outs[0], outs[2], tol)


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_incremental_prefill_equals_one_shot(golden, dtype, tol):
    """Prefilling the query in two pieces on the same context gives the one-shot logits (incremental == one-shot,
    proj/tests/test_model.cpp:175-194), and the context grows to the same length and next position."""
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], dtype)
    ids = eng.ingest_chunks(payloads(A, "c1"))
    q = A["c1.query"]
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        one = eng.prefill_query(ctx, q)[0]
        n_one, p_one = ctx.total_tokens(), ctx.next_position
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        eng.prefill_query(ctx, q[:13])
        two = eng.prefill_query(ctx, q[13:])[0]
        assert (ctx.total_tokens(), ctx.next_position) == (n_one, p_one)
    assert_close(two, one, tol)


def test_tkvc_export_loads_in_reference(golden, tmp_path):
    """Chunks precomputed on the GPU (f32) exported as TKVC files are loaded by the UNMODIFIED reference
    CacheStore (header, offsets, fingerprint, dims validated, kvstore.cpp:134-207) and its assemble + query
    prefill over them matches its own recomputed caches within fp32 rounding."""
    if not O.Ref.available():
        pytest.skip("reference sources absent (GPU box)")
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], "f32")
    pays = payloads(A, "c1")
    ids = eng.ingest_chunks(pays)
    ref_gpu = O.RefEngine(O.TOY, m["seed"], str(tmp_path / "from_gpu"), f32_store=True)
    ref_own = O.RefEngine(O.TOY, m["seed"], str(tmp_path / "own"), f32_store=True)
    try:
        assert ref_gpu.fingerprint() == eng.fingerprint()
        for cid in ids:
            path = ref_gpu.store_path(cid)
            os.makedirs(os.path.dirname(path), exist_ok=True)
            eng.export_tkvc(cid, path)
        assert [ref_own.ingest(p) for p in pays] == ids
        q = A["c1.query"]
        got, _ = ref_gpu.assemble(ids, True).prefill_query(q)
        want, _ = ref_own.assemble(ids, True).prefill_query(q)
        assert_close(got, want, FP32_TOL)
    finally:
        ref_gpu.close()
        ref_own.close()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_rope_position_zero_is_identity(golden, dtype):
    """RoPE at position 0 is the bit-exact identity (proj/tests/test_rope.cpp:42-52): the gathered, rotated key of
    the context's first token equals its unrotated row bitwise, in every layer."""
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], dtype)
    ids = eng.ingest_chunks(payloads(A, "c1"))
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        assert ctx.positions[0] == 0
        for layer in range(cfg_t(m).layer_num):
            assert np.array_equal(ctx.read_kv(layer, "k", rotated=True)[0], ctx.read_kv(layer, "k", rotated=False)[0])


def test_layer0_kv_is_position_free(golden):
    """Layer-0 K/V (unrotated) depend only on the token, not on its position (proj/tests/test_model.cpp:157-173):
    a chunk's stored layer-0 rows equal its rows inside a full-concat forward where it sits behind another chunk."""
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], "f32")
    pay = payloads(A, "c1")[:2]
    ids = eng.ingest_chunks(pay)
    framed = [O.frame(p) for p in pay]
    with eng.naive_prefill(framed, A["c1.query"], T.MaskMode.Causal) as ctx:
        k0 = ctx.read_kv(0, "k", rotated=False)
        v0 = ctx.read_kv(0, "v")
    n0 = len(framed[0])
    for which, full in (("k", k0), ("v", v0)):
        assert np.allclose(eng.store_read(ids[1], 0, which), full[n0:n0 + len(framed[1])], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_tkvc_import_gather_bit_exact(golden, tmp_path, dtype):
    """Reference-format chunk caches -> HBM store -> fused gather: unrotated pages bit-exact after the
    canonical cast, rotated keys within fp32 rounding of rope(ctx.k, positions)."""
    meta, A = golden
    m = meta["c1"]
    cfg = O.TOY
    framed = [O.frame(p) for p in payloads(A, "c1")]
    paths, kvs = [], []
    fresh_seed = 4242 + (dtype == "bf16")
    port2 = O.Port(cfg, fresh_seed)
    eng2 = T.Engine(cfg_t(m), fresh_seed, dtype=dtype, store_capacity_tokens=4096)
    for f in framed:
        k, v = port2.chunk_kv(f)
        kvs.append((k, v))
        paths.append(write_tkvc(str(tmp_path), port2.chunk_id(f), port2.fingerprint(), k, v, cfg.kv_head_num,
                                cfg.head_size))
    ids = [eng2.import_tkvc(p) for p in paths]
    assert ids == [port2.chunk_id(f) for f in framed]
    cast = (lambda x: x.astype(np.float32)) if dtype == "f32" else to_bf16
    for (k, v), cid in zip(kvs, ids):
        for layer in range(cfg.layer_num):
            assert np.array_equal(eng2.store_read(cid, layer, "k"), cast(k[layer]))
            assert np.array_equal(eng2.store_read(cid, layer, "v"), cast(v[layer]))
    for mode in (T.PositionMode.Reordered, T.PositionMode.Composite):
        with eng2.assemble(ids, mode) as ctx:
            kref, vref, pos, nxt = port2.assemble(framed, mode == T.PositionMode.Reordered)
            assert np.array_equal(ctx.positions, pos) and ctx.next_position == nxt
            for layer in (0, cfg.layer_num - 1):
                assert np.array_equal(ctx.read_kv(layer, "k", rotated=False), cast(kref[layer]))
                assert np.array_equal(ctx.read_kv(layer, "v"), cast(vref[layer]))
                rot_ref = O.Port.rope(cast(kref[layer]).astype(np.float64), pos, cfg.head_size)
                rot = ctx.read_kv(layer, "k", rotated=True)
                atol = 1e-6 if dtype == "f32" else 8e-3
                assert np.abs(rot - rot_ref).max() <= atol * max(1.0, np.abs(rot_ref).max())
            logits = eng2.prefill_query(ctx, A["c1.query"])[0]
            ref = port2.prefill_query(kref, vref, pos, nxt, A["c1.query"])
            assert_close(logits, ref, FP32_TOL if dtype == "f32" else BF16_TOL)
    eng2.close()


def dense(lo, hi, cols):
    j = np.arange(cols)[None, :]
    return ((j >= np.asarray(lo)[:, None]) & (j <= np.asarray(hi)[:, None])).astype(np.uint8)


def test_masks_bit_exact(golden):
    """The [lo, hi] predicate the kernels apply, materialised on device, equals the reference masks."""
    meta, A = golden
    eng = engine(T.ModelConfig.toy(), 42, "f32")
    framed = [O.frame([97] * n) for n in (1, 2, 3)]  # framed lengths 3, 4, 5
    q = [98, 99]
    for mode, tag in ((T.MaskMode.Causal, "causal"), (T.MaskMode.Independent, "independent")):
        with eng.naive_prefill(framed, q, mode) as ctx:
            assert np.array_equal(ctx.mask(14, 14), A[f"mask.3452.{tag}"])
    ids = eng.ingest_chunks([[97], [98, 99]])  # framed 3 + 4 = 7 past tokens
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        eng.prefill_query(ctx, [100, 101, 102, 103, 104])
        assert np.array_equal(ctx.mask(5, 12), A["mask.causal_rows_5_7"])


def test_positions_345(golden):
    meta, _ = golden
    eng = engine(T.ModelConfig.toy(), 42, "f32")
    ids = eng.ingest_chunks([T.encode(s) for s in ("a", "bc", "def")])
    for mode, tag in ((T.PositionMode.Reordered, "reordered"), (T.PositionMode.Composite, "composite")):
        with eng.assemble(ids, mode) as ctx:
            assert ctx.positions.tolist() == meta[f"positions_345.{tag}"]["positions"]
            assert ctx.next_position == meta[f"positions_345.{tag}"]["next"]
            assert ctx.segments == [(3, "chunk"), (4, "chunk"), (5, "chunk")]
    with eng.assemble([], T.PositionMode.Reordered) as ctx:
        assert ctx.total_tokens() == 0 and ctx.next_position == 0


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_ingest_kv_matches_oracle(dtype):
    """Offline block-diagonal chunk prefill (several chunks packed in one forward) vs ingest_chunk_payload."""
    cfg = O.TOY
    port = O.Port(cfg, 42)
    eng = engine(T.ModelConfig.toy(), 42, dtype)
    pays = [O.random_text_tokens(9000 + i, n) for i, n in enumerate((5, 70, 1, 129))]
    ids = eng.ingest_chunks(pays)
    tol = 1e-4 if dtype == "f32" else 2e-2
    for p, cid in zip(pays, ids):
        k, v = port.chunk_kv(O.frame(p))
        for layer in range(cfg.layer_num):
            assert_close(eng.store_read(cid, layer, "k"), k[layer], tol)
            assert_close(eng.store_read(cid, layer, "v"), v[layer], tol)


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_qwen_dims_one_layer_vs_golden(golden, dtype, tol):
    meta, A = golden
    m = meta["qwen1"]
    eng = engine(cfg_t(m), m["seed"], dtype)
    assert f"{eng.fingerprint():016x}" == m["fingerprint"]
    ids = eng.ingest_chunks(payloads(A, "qwen1"))
    assert [f"{i:016x}" for i in ids] == m["ids"]
    for mode, tag in ((T.PositionMode.Reordered, "reordered"), (T.PositionMode.Composite, "composite")):
        with eng.assemble(ids, mode) as ctx:
            logits = eng.prefill_query(ctx, A["qwen1.query"])[0]
            assert_close(logits, A[f"qwen1.turbo_{tag}.logits"], tol)
            assert_argmax(logits, A[f"qwen1.turbo_{tag}.logits"], tol)
    framed = [O.frame(p) for p in payloads(A, "qwen1")]
    for mode, tag in ((T.MaskMode.Causal, "causal"), (T.MaskMode.Independent, "independent")):
        assert_close(eng.naive_prefill(framed, A["qwen1.query"], mode, keep_context=False)[0],
                     A[f"qwen1.naive_{tag}.logits"], tol)


def test_decode_attention_flag_vs_golden(golden):
    """TKV_FLAG_DECODE_ATTN: the last layer's single row (query prefill) and every greedy-decode step run the
    decode-sized split-K kernel (R = 7 rows per kv head at Qwen dims); logits within bf16 tolerance of the
    golden and of the default tcgen05 path, same greedy tokens."""
    meta, A = golden
    m = meta["qwen1"]
    dec = engine(cfg_t(m), m["seed"], "bf16", flags=0x40)
    ref = engine(cfg_t(m), m["seed"], "bf16")
    outs = []
    for eng in (dec, ref):
        ids = eng.ingest_chunks(payloads(A, "qwen1"))
        with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
            logits = eng.prefill_query(ctx, A["qwen1.query"])[0]
            assert_close(logits, A["qwen1.turbo_reordered.logits"], BF16_TOL)
            outs.append((logits, eng.greedy_decode(ctx, 4)))
    assert_close(outs[0][0], outs[1][0], BF16_TOL)
    assert outs[0][1] == outs[1][1]


def test_tcgen05_gemm_matches_simt_gemm():
    """bf16 tcgen05/TMA GEMM vs the SIMT GEMM on the same bf16 inputs (exact Qwen dims, 2 layers)."""
    cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
    tc = engine(cfg, 7, "bf16")
    simt = engine(cfg, 7, "bf16", flags=T.FLAG_SIMT_GEMM)
    pays = [O.random_text_tokens(500 + i, 254) for i in range(6)]
    q = O.random_text_tokens(501, 64)
    outs = []
    for eng in (tc, simt):
        ids = eng.ingest_chunks(pays)
        with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
            outs.append(eng.prefill_query(ctx, q)[0])
        outs.append(eng.naive_prefill([O.frame(p) for p in pays], q, T.MaskMode.Causal, keep_context=False)[0])
    assert_close(outs[0], outs[2], 1e-2)
    assert_close(outs[1], outs[3], 1e-2)


def test_greedy_decode_matches_reference(golden):
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], "f32")
    ids = eng.ingest_chunks(payloads(A, "c1"))
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        eng.prefill_query(ctx, A["c1.query"])
        assert eng.greedy_decode(ctx, 8) == m["decode8"]


def test_errors_map_to_reference_classes(tmp_path):
    eng = engine(T.ModelConfig.toy(), 42, "f32")
    ids = eng.ingest_chunks([[97, 98]])
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        with pytest.raises(T.DomainError):
            eng.prefill_query(ctx, [])
        with pytest.raises(T.DomainError):
            eng.prefill_query(ctx, [300])
    with pytest.raises(T.NotFoundError):
        eng.assemble([0x1234], T.PositionMode.Reordered)
    with pytest.raises(T.DomainError):
        eng.naive_prefill([[256, 257], []], [97], T.MaskMode.Causal)
    with pytest.raises(T.ConfigError):
        T.Engine(T.ModelConfig(4, 8, 3, 8, 64, 192, 259), 1)
    # a cache built under another model is stale (kvstore.cpp:169-172)
    port = O.Port(O.TOY, 43)
    f = O.frame([97, 98])
    k, v = port.chunk_kv(f)
    p = write_tkvc(str(tmp_path), port.chunk_id(f), port.fingerprint(), k, v, 2, 8)
    with pytest.raises(T.StaleCacheError):
        eng.import_tkvc(p)
    # same model, damaged file: FormatError (fingerprint is checked before the size, kvstore.cpp:169-191)
    port42 = O.Port(O.TOY, 42)
    k, v = port42.chunk_kv(f)
    good = write_tkvc(str(tmp_path), port42.chunk_id(f), port42.fingerprint(), k, v, 2, 8)
    raw = open(good, "rb").read()
    bad = tmp_path / "trunc.tkvc"
    bad.write_bytes(raw[:-8])
    with pytest.raises(T.FormatError):
        eng.import_tkvc(str(bad))
    with pytest.raises(T.NotFoundError):
        eng.import_tkvc(str(tmp_path / "missing.tkvc"))


def test_mask_fault_breaks_equivalence(golden):
    """verify --inject-fault (tools/turbokv_main.cpp:593-599): a corrupted independent mask must show."""
    meta, A = golden
    eng = engine(T.ModelConfig.toy(), 42, "f32")
    framed = [O.frame(p) for p in payloads(A, "c1")]
    q = A["c1.query"]
    clean = eng.naive_prefill(framed, q, T.MaskMode.Independent, keep_context=False)[0]
    eng.set_mask_fault(200, 0)  # a row of chunk 1 may now see chunk 0
    faulty = eng.naive_prefill(framed, q, T.MaskMode.Independent, keep_context=False)[0]
    assert np.abs(faulty - clean).max() > 1e-6


@pytest.mark.skipif(not O.Ref.available(), reason="reference library not built")
@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_inject_fault_reproduces_reference(golden, dtype, tol, tmp_path):
    """The reference's exact `verify --inject-fault` corruption (tools/turbokv_main.cpp:593-599: the last query row
    loses column 0, through testing::mask_fault_hook) on both sides: the faulty naive-independent logits of this
    engine equal the UNMODIFIED reference's faulty logits, and differ from the clean ones."""
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], dtype)
    framed = [O.frame(p) for p in payloads(A, "c1")]
    q = A["c1.query"]
    n = sum(len(f) for f in framed) + len(q)
    eng.set_mask_rows([-1], [1], [n - 1])
    faulty = eng.naive_prefill(framed, q, T.MaskMode.Independent, keep_context=False)[0]
    ref_eng = O.RefEngine(O.Cfg(**m["config"]), m["seed"], str(tmp_path))
    O.Ref.check(O.Ref.lib().ref_set_inject_fault(1))
    try:
        ref_faulty = ref_eng.naive_prefill(framed, q, True)
    finally:
        O.Ref.check(O.Ref.lib().ref_set_inject_fault(0))
        ref_eng.close()
    assert_close(faulty, ref_faulty, tol)
    clean = A["c1.naive_independent.logits"]
    assert np.abs(ref_faulty - clean).max() > 1e-3  # the fault is visible in the reference itself
    assert np.abs(faulty.astype(np.float64) - clean).max() > 1e-3


def test_gather_roundtrip_at_c2_chunk_shape():
    """Size-independent properties at the C2 chunk shape (Qwen dims, 16 x 512-token chunks, 2 layers):
    the identity gather reproduces the store bit for bit, and rotated rows equal R(pos) applied to them."""
    cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
    eng = engine(cfg, 11, "bf16")
    pays = [O.random_text_tokens(700 + i, 510) for i in range(16)]
    ids = eng.ingest_chunks(pays)
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        assert ctx.total_tokens() == 16 * 512 and ctx.next_position == 8192
        unrot = ctx.read_kv(1, "k", rotated=False)
        rot = ctx.read_kv(1, "k", rotated=True)
        v = ctx.read_kv(1, "v")
        stored_k = np.concatenate([eng.store_read(i, 1, "k") for i in ids])
        stored_v = np.concatenate([eng.store_read(i, 1, "v") for i in ids])
        assert np.array_equal(unrot, stored_k) and np.array_equal(v, stored_v)
        rows = np.r_[0:64, 4000:4064, 8128:8192]
        ref = O.Port.rope(stored_k[rows].astype(np.float64), ctx.positions[rows], cfg.head_size)
        assert np.abs(rot[rows] - ref).max() <= 8e-3 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("policy", ["direct", "fetch"])
def test_remote_chunks_gathered_from_peer_pool(policy):
    """Two engines (two shards); engine A serves a request whose chunks live partly in B's pool: the gather
    kernel reads B's pages through the peer pool table (or after a fetch-once copy). The logits must equal
    a single engine holding every chunk locally, bit for bit."""
    cfg = T.ModelConfig.toy()
    a = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=4096)
    b = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=4096)
    whole = engine(cfg, 42, "bf16")
    pays = [O.random_text_tokens(8800 + i, n) for i, n in enumerate((70, 5, 130, 64))]
    ids = whole.ingest_chunks(pays)
    assert a.ingest_chunks([pays[0], pays[2]]) == [ids[0], ids[2]]
    assert b.ingest_chunks([pays[1], pays[3]]) == [ids[1], ids[3]]
    a.attach_engine(1, b)
    for i in (1, 3):
        pages, length = b.chunk_pages(ids[i])
        a.register_remote(ids[i], 1, length, pages, O.frame(pays[i]))
    if policy == "fetch":
        for i in (1, 3):
            a.fetch_remote(ids[i])
    q = O.random_text_tokens(8899, 21)
    with whole.assemble(ids, T.PositionMode.Reordered) as c0, a.assemble(ids, T.PositionMode.Reordered) as c1:
        ref = whole.prefill_query(c0, q)
        got = a.prefill_query(c1, q)
        assert np.array_equal(got, ref)
        assert np.array_equal(c1.read_kv(2, "v"), c0.read_kv(2, "v"))
    per_token = cfg.layer_num * 2 * cfg.kv_dim * 2  # K and V, bf16
    if policy == "direct":  # the 7- and 66-token chunks were read over the peer pool by one gather
        assert a.remote_bytes() == (7 + 66) * per_token
    else:  # copied once, page by page (1 + 2 pages of 64 tokens)
        assert a.remote_bytes() == 3 * 64 * per_token
    a.close()
    b.close()


@pytest.mark.gpu
def test_store_evict_reuses_pages_and_guards_stale_reads():
    cfg = T.ModelConfig.toy()
    eng = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=512)
    payloads = [O.random_text_tokens(3000 + i, 126) for i in range(3)]
    ids = eng.ingest_chunks(payloads)
    n0, used0, total = eng.store_count()
    ctx = eng.assemble(ids[:2], T.PositionMode.Reordered)
    before = eng.prefill_query(ctx, O.random_text_tokens(7, 16))[0]
    eng.store_evict(ids[0])
    assert not eng.store_contains(ids[0]) and eng.store_contains(ids[1])
    assert eng.store_count()[1] == used0 - 2  # a 128-token chunk owns two 64-token pages
    with pytest.raises(T.StaleCacheError):
        ctx.read_kv(0, "k", rotated=False)
    ctx.read_kv(0, "k", rotated=True)  # the gathered cache itself is unaffected
    with pytest.raises(T.NotFoundError):
        eng.store_evict(ids[0])
    with pytest.raises(T.NotFoundError):
        eng.assemble(ids[:1], T.PositionMode.Reordered)
    # re-ingest: same content id, pages reused; logits agree to bf16 tolerance (a lone 128-token chunk takes
    # the swapped GEMM tiling, the original 3-chunk batch the normal one: different fp32 summation order)
    assert eng.ingest_chunks(payloads[:1])[0] == ids[0]
    ctx2 = eng.assemble(ids[:2], T.PositionMode.Reordered)
    after = eng.prefill_query(ctx2, O.random_text_tokens(7, 16))[0]
    assert np.abs(before - after).max() <= 2e-2 * np.abs(before).max()
    ctx.close()
    ctx2.close()
    eng.close()


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("name", ["c1", "ragged", "qwen1"])
def test_batched_prefill_vs_golden(golden, name, dtype, tol):
    """tkv_prefill_query_batch (C3's batched path): a reordered and a composite context of the same chunks in ONE
    forward, each against the reference's logits, plus a third request over a chunk subset against the same
    engine's single-request prefill; context bookkeeping identical to prefill_query."""
    meta, A = golden
    m = meta[name]
    eng = engine(cfg_t(m), m["seed"], dtype)
    ids = eng.ingest_chunks(payloads(A, name))
    q = A[f"{name}.query"]
    ctxs = [eng.assemble(ids, T.PositionMode.Reordered), eng.assemble(ids, T.PositionMode.Composite),
            eng.assemble(ids[::-1][:max(1, len(ids) - 1)], T.PositionMode.Reordered)]
    q3 = np.asarray(q[: max(1, len(q) // 2)])
    logits = eng.prefill_query_batch(ctxs, [q, q, q3])
    for r, tag in ((0, "reordered"), (1, "composite")):
        ref = A[f"{name}.turbo_{tag}.logits"]
        assert_close(logits[r], ref, tol)
        assert_argmax(logits[r], ref, tol)
        assert ctxs[r].total_tokens() == len(ctxs[r].positions)
        assert ctxs[r].next_position == m[f"{tag}.next_position"] + len(q)
    with eng.assemble(ids[::-1][:max(1, len(ids) - 1)], T.PositionMode.Reordered) as single:
        ref3 = eng.prefill_query(single, q3)[0]
        assert_close(logits[2], ref3, tol)
        assert np.array_equal(single.positions, ctxs[2].positions)
    for c in ctxs:
        c.close()


def test_batched_prefill_rejects_bad_batches(golden):
    meta, A = golden
    m = meta["c1"]
    eng = engine(cfg_t(m), m["seed"], "bf16")
    ids = eng.ingest_chunks(payloads(A, "c1"))
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        with pytest.raises(T.ConfigError):
            eng.prefill_query_batch([ctx, ctx], [A["c1.query"], A["c1.query"]])
        with pytest.raises(T.DomainError):
            eng.prefill_query_batch([ctx], [np.zeros(0, np.int32)])



@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_host_spill_tier_is_bit_exact_and_transparent(golden, dtype):
    """Chunks that do not fit the HBM store land in the pinned host tier: ingest writes their pages over the
    mapped host pointer, the gather kernel reads them zero-copy; pages, gathered KV and logits are identical
    to an all-HBM engine (north star subsystem 1: HBM store + pinned host when it spills)."""
    meta, A = golden
    m = meta["c1"]
    cfg = cfg_t(m)
    ref = engine(cfg, m["seed"], dtype)
    spill = T.Engine(cfg, m["seed"], dtype=dtype, store_capacity_tokens=256, host_spill_tokens=1024)
    pl = payloads(A, "c1")
    ids_ref, ids = ref.ingest_chunks(pl), spill.ingest_chunks(pl)
    assert ids == ids_ref
    tiers = [spill.store_chunk_tier(i) for i in ids]
    assert tiers[:2] == [0, 0] and tiers[2:] == [1, 1]  # 2 x 128 tokens fill the 256-token HBM store
    t = spill.store_tiers()
    assert t["hbm_used"] == t["hbm_total"] == 4 and t["host_used"] == 4 and t["host_total"] == 16
    for i in ids:
        for layer in (0, cfg.layer_num - 1):
            for which in ("k", "v"):
                assert np.array_equal(spill.store_read(i, layer, which), ref.store_read(i, layer, which))
    q = A["c1.query"]
    with spill.assemble(ids, T.PositionMode.Reordered) as c1, ref.assemble(ids, T.PositionMode.Reordered) as c0:
        for layer in (0, cfg.layer_num - 1):
            assert np.array_equal(c1.read_kv(layer, "k", rotated=True), c0.read_kv(layer, "k", rotated=True))
            assert np.array_equal(c1.read_kv(layer, "v"), c0.read_kv(layer, "v"))
        assert np.array_equal(spill.prefill_query(c1, q)[0], ref.prefill_query(c0, q)[0])
    spill.store_evict(ids[2])
    assert spill.store_tiers()["host_used"] == 2
    spill.close()



@pytest.mark.parametrize("name", ["qwen1"])
def test_batched_attention_single_launch_vs_golden(golden, name):
    """The batched prefill's single attention launch over every request's cache (3-D tensor maps; the C3 path),
    forced on a small batch, against the reference's logits and the per-request path."""
    meta, A = golden
    m = meta[name]
    eng = engine(cfg_t(m), m["seed"], "bf16", flags=0x20)  # TKV_FLAG_BATCH_ATTN
    ids = eng.ingest_chunks(payloads(A, name))
    q = A[f"{name}.query"]
    ctxs = [eng.assemble(ids, T.PositionMode.Reordered), eng.assemble(ids, T.PositionMode.Composite),
            eng.assemble(ids[:1], T.PositionMode.Reordered)]
    q3 = np.asarray(q[:5])
    logits = eng.prefill_query_batch(ctxs, [q, q, q3])
    for r, tag in ((0, "reordered"), (1, "composite")):
        ref = A[f"{name}.turbo_{tag}.logits"]
        assert_close(logits[r], ref, BF16_TOL)
        assert_argmax(logits[r], ref, BF16_TOL)
    with eng.assemble(ids[:1], T.PositionMode.Reordered) as single:
        assert_close(logits[2], eng.prefill_query(single, q3)[0], BF16_TOL)
    for c in ctxs:
        c.close()


def test_index_top_k_matches_reference():
    """GPU cosine top-k (retrieval.cu) over a 3000-chunk index: ids AND cosines bit-identical to the reference's
    RetrievalIndex::top_k, incl. exact ties (same payload under two ids -> ascending id) and k > size."""
    cfg = T.ModelConfig.toy()
    eng = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=4096)
    rng = np.random.default_rng(11)
    payloads = [O.random_text_tokens(20000 + i, int(rng.integers(1, 200))) for i in range(3000)]
    ids = [int(x) for x in np.unique(rng.integers(1, 1 << 40, 3100, dtype=np.int64))[:3000]]
    rng.shuffle(ids)
    for i, p in zip(ids, payloads):
        assert eng.index_add(i, p)
    twin = ids[17] + 1 if ids[17] + 1 not in ids else ids[17] - 1
    assert eng.index_add(twin, payloads[17])       # exact cosine tie with ids[17]
    assert not eng.index_add(ids[5], payloads[5])  # content dedup by id
    ingested = eng.ingest_chunks([O.random_text_tokens(99, 126)])  # auto-indexed by ingest
    assert eng.index_size() == 3002
    all_ids = np.array(ids + [twin, ingested[0]], np.uint64)
    emb = np.stack([O.Port.embed(p) for p in payloads + [payloads[17], O.random_text_tokens(99, 126)]])
    for qs, k in ((1, 1), (2, 16), (3, 100), (4, 256)):
        q = O.random_text_tokens(40000 + qs, 60) if qs != 4 else payloads[17]
        got, scores = eng.top_k(q, k)
        ref_ids, ref_scores = O.Port.top_k(emb, all_ids, O.Port.embed(q), k)
        assert np.array_equal(got, ref_ids)
        assert np.array_equal(scores, ref_scores)
        if qs == 1:
            assert np.array_equal(got, O.Ref.top_k(emb, all_ids, O.Port.embed(q), k))
    small = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=1024)
    small.index_add(5, payloads[0])
    small.index_add(3, payloads[1])
    got, _ = small.top_k(payloads[1], 10)  # k beyond the index size returns everything
    assert list(got) == [3, 5]
    with pytest.raises(T.DomainError):
        small.top_k(payloads[1], 0)
    small.close()
    eng.close()


_TILING_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import oracle as O
from paper_2410_07590_b200 import turbokv as T
cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
eng = T.Engine(cfg, 7, dtype="bf16", store_capacity_tokens=1 << 16)
pays = [O.random_text_tokens(700 + i, 510) for i in range(5)]
q = O.random_text_tokens(701, 64)
out = eng.naive_prefill([O.frame(p) for p in pays], q, T.MaskMode.Causal, keep_context=False)[0]
np.save(sys.argv[1], out)
"""


@pytest.mark.parametrize("env", [{"TKV_GEMM_NSMP": "1", "TKV_GEMM_RASTER": "0"}])
def test_large_m_gemm_tilings_agree(tmp_path, env):
    """The large-M (> 128 tokens) GEMM variant with one 128-row activation tile per unit and n-fastest raster gives
    the default tiling's full-concat logits (bf16 tolerance); each runs in a fresh process because the tiling knobs
    are process-wide (read from the environment by TUNING builds; a release library runs the default twice)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "run.py"
    script.write_text(_TILING_SCRIPT.format(root=root))
    outs = []
    for e in ({}, env):
        path = tmp_path / f"out{len(outs)}.npy"
        subprocess.run([sys.executable, str(script), str(path)], check=True, env={**os.environ, **e}, timeout=300)
        outs.append(np.load(path))
    assert_close(outs[1], outs[0], BF16_TOL)


def test_batched_attention_split_k_matches():
    """The batched single-launch attention with split-K partials and the request-aware combine: 10 requests x
    (3 x 800-token chunks + a 64-token query) give 160 (request, kv head, row tile) CTAs, for which the automatic
    split picker (attn_tc_batch_pick_splits) chooses 2 splits to fill the last wave; every request's logits equal its
    own prefill_query (bf16 tolerance, argmax checked)."""
    cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
    eng = engine(cfg, 7, "bf16", flags=0x20)  # TKV_FLAG_BATCH_ATTN
    ids = eng.ingest_chunks([O.random_text_tokens(800 + i, 798) for i in range(12)])
    picks = [[ids[(r + k) % 12] for k in range(3)] for r in range(10)]
    qs = [O.random_text_tokens(860 + r, 64) for r in range(10)]
    ctxs = [eng.assemble(p) for p in picks]
    eng.kernel_timeline(True)
    batched = eng.prefill_query_batch(ctxs, qs)
    _, cls = eng.kernel_timeline(False)
    assert (cls == T.Engine.TIMELINE_CLASSES.index("attention")).sum() == 2 * cfg.layer_num  # attention + split merge
    for c in ctxs:
        c.close()
    for r in (0, 4, 9):
        with eng.assemble(picks[r]) as single:
            ref = eng.prefill_query(single, qs[r])[0]
        assert_close(batched[r], ref, BF16_TOL)
        assert_argmax(batched[r], ref, BF16_TOL)


def test_batched_prefill_many_tokens_matches_per_request():
    """A batched forward above 256 query tokens (the per-token-row QKV epilogue writing every request's K/V to its
    own cache through the request table, many-token residuals, the single batched attention launch with its
    automatic split-K) gives each request the logits of its own prefill_query, and leaves the same query K/V rows
    in its cache (Qwen dims, 2 layers; bf16 tolerance, argmax checked)."""
    cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
    eng = engine(cfg, 7, "bf16", flags=0x20)  # TKV_FLAG_BATCH_ATTN: one attention launch for the batch
    ids = eng.ingest_chunks([O.random_text_tokens(900 + i, 300 + 37 * i) for i in range(8)])
    qs = [O.random_text_tokens(950 + r, 48 + 3 * r) for r in range(6)]
    assert sum(len(q) for q in qs) > 256
    picks = [ids[r:r + 3] for r in range(6)]
    ctxs = [eng.assemble(p, T.PositionMode.Reordered if r % 2 else T.PositionMode.Composite)
            for r, p in enumerate(picks)]
    batched = eng.prefill_query_batch(ctxs, qs)
    for r, (p, q) in enumerate(zip(picks, qs)):
        with eng.assemble(p, T.PositionMode.Reordered if r % 2 else T.PositionMode.Composite) as single:
            ref = eng.prefill_query(single, q)[0]
            assert_close(batched[r], ref, BF16_TOL)
            assert_argmax(batched[r], ref, BF16_TOL)
            for layer in (0, cfg.layer_num - 1):
                n = single.total_tokens()
                kb = ctxs[r].read_kv(layer, "k", rotated=True)[n - len(q):n]
                ks = single.read_kv(layer, "k", rotated=True)[n - len(q):n]
                assert_close(kb, ks, BF16_TOL)
    for c in ctxs:
        c.close()


def test_kernel_timeline_covers_the_forward():
    """tkv_kernel_timeline: every hot launch of a query prefill is stamped in stream order with its class (one gather,
    embed, 4 GEMMs + QKV epilogue + attention (+ merge) + 2 residuals per layer, lm_head), every duration is
    positive, the launches do not overlap out of order, and disarming leaves later launches unstamped."""
    cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
    eng = engine(cfg, 5, "bf16")
    ids = eng.ingest_chunks([O.random_text_tokens(700 + i, 200) for i in range(3)])
    q = O.random_text_tokens(77, 33)
    eng.kernel_timeline(True)
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        eng.prefill_query(ctx, q)
    tl, cls = eng.kernel_timeline(False)
    names = [T.Engine.TIMELINE_CLASSES[c] for c in cls]
    assert names[0] == "gather_rope" and names[1] == "epilogue" and names[-1] == "other"
    assert names.count("gemm") == 4 * cfg.layer_num
    assert names.count("epilogue") == 1 + 3 * cfg.layer_num
    assert cfg.layer_num <= names.count("attention") <= 2 * cfg.layer_num
    assert (tl[:, 1] > tl[:, 0]).all() and (tl[:, 0] > 0).all()
    assert (np.diff(tl[:, 1]) > 0).all()  # each launch finishes after its predecessor (stream order)
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        eng.prefill_query(ctx, q)
    tl2, _ = eng.kernel_timeline(False)
    assert len(tl2) == 0


def test_graph_replay_is_bitwise_the_kernel_chain():
    """CUDA-graph replay of the query-prefill forward (captured on the second forward with the same shape and
    buffers, replayed afterwards) gives bitwise the logits and cache rows of the kernel-by-kernel chain
    (TKV_FLAG_NO_GRAPHS), over recycled contexts, device-token prefill, a changed query, and a different chunk order
    of the same length (same graph key: the cache contents and positions change under the captured pointers)."""
    import torch
    cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
    outs = {}
    for flags in (0, T.FLAG_NO_GRAPHS):
        eng = engine(cfg, 5, "bf16", flags=flags)
        ids = eng.ingest_chunks([O.random_text_tokens(700 + i, 300) for i in range(4)])
        res = []
        for rep in range(4):
            q = O.random_text_tokens(90 + (rep // 3), 40)  # the 4th request changes the query tokens
            with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
                res.append(eng.prefill_query(ctx, q)[0].copy())
                res.append(ctx.read_kv(1, "k", rotated=True)[-40:].copy())
        dq = torch.from_numpy(O.random_text_tokens(91, 40)).cuda()
        dl = torch.empty(cfg.vocab_size, dtype=torch.float32, device="cuda")
        for rep in range(4):
            order = ids if rep < 3 else ids[::-1]  # the 4th request: same length, other chunk order
            with eng.assemble(order, T.PositionMode.Reordered) as ctx:
                eng.prefill_query_device(ctx, dq.data_ptr(), 40, dl.data_ptr())
                eng.check()
                res.append(dl.cpu().numpy().copy())
        outs[flags] = res
        eng.close()
    assert not np.array_equal(outs[0][-1], outs[0][-2])  # the reordered context really changed the logits
    for a, b in zip(outs[0], outs[T.FLAG_NO_GRAPHS]):
        assert np.array_equal(a, b)
