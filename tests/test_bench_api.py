"""The reference's bench API mirror (paper_2410_07590_b200/bench_api.py vs proj/src/bench.cpp).

CPU: the bench corpus is the reference's own (chunk ids equal to those of the UNMODIFIED reference's
ingest_synthetic), the CSV/summary formats and the validation errors. GPU: run_bench on exact Qwen2-7B dims
(2 layers) -- one row per (grid point, path, rep), FlopCounter totals equal to the reference cost model, and the
reference acceptance criterion (acceptance_main.cpp:296-329): speedup monotone over the grid, >= 3x at 4096.
"""
import numpy as np
import pytest

import oracle as O
from paper_2410_07590_b200 import bench_api as B
from paper_2410_07590_b200 import turbokv as T


def test_splitmix_stream_matches_reference_at():
    rng = B.SplitMix64(42)
    assert [rng.next() for _ in range(5)] == [O.splitmix_at(42, i) for i in range(5)]


@pytest.mark.parametrize("grid,seed", [([64, 192], 42), ([128, 512, 320], 7)])
def test_corpus_chunk_ids_equal_reference_ingest_synthetic(tmp_path, grid, seed):
    payloads = B.synthetic_payloads(B.BenchConfig(doc_grid=grid, seed=seed))
    assert len(payloads) == max(grid) // 64 and all(len(p) == 62 for p in payloads)
    port = O.Port(O.TOY, 42)
    ours = [port.chunk_id(O.frame(p)) for p in payloads]
    if not O.Ref.available():
        pytest.skip("reference sources absent (GPU box)")
    ref = O.RefEngine(O.TOY, 42, str(tmp_path / "store"))
    try:
        assert ours == ref.bench_ingest(grid, seed)
    finally:
        ref.close()


def test_query_is_seeded_letters():
    q = B.bench_query(B.BenchConfig(doc_grid=[64], query_tokens=64, seed=42))
    assert len(q) == 64 and ((q >= 97) & (q <= 122)).all()
    assert np.array_equal(q, B.bench_query(B.BenchConfig(doc_grid=[128], query_tokens=64, seed=42)))


def test_csv_and_summary_formats():
    rows = [B.BenchRow(64, 8, "turbo-reordered", 0, 12.3456789, 100), B.BenchRow(64, 8, "turbo-reordered", 1, 0.5, 100),
            B.BenchRow(64, 8, "naive-independent", 0, 1234567.0, 900),
            B.BenchRow(64, 8, "naive-independent", 1, 3.0, 900)]
    csv = B.bench_csv(rows).splitlines()
    assert csv[0] == "doc_tokens,query_tokens,path,rep,ttft_ms,measured_flops"
    assert csv[1:] == ["64,8,turbo-reordered,0,12.3457,100", "64,8,turbo-reordered,1,0.5,100",
                       "64,8,naive-independent,0,1.23457e+06,900", "64,8,naive-independent,1,3,900"]
    (s,) = B.summarize(rows)
    assert s.doc_tokens == 64 and s.turbo_median_ms == pytest.approx((12.3456789 + 0.5) / 2)
    assert s.naive_median_ms == pytest.approx((1234567.0 + 3.0) / 2)
    assert s.speedup == pytest.approx(s.naive_median_ms / s.turbo_median_ms)
    with pytest.raises(T.DomainError):
        B.summarize(rows[:2])


@pytest.mark.parametrize("cfg", [B.BenchConfig(doc_grid=[]), B.BenchConfig(doc_grid=[63]),
                                 B.BenchConfig(doc_grid=[0])])
def test_grid_validation(cfg):
    with pytest.raises(T.DomainError):
        B.synthetic_payloads(cfg)


@pytest.mark.gpu
def test_run_bench_qwen_dims_rows_flops_and_acceptance():
    cfg = T.ModelConfig(**vars(O.qwen_layers(2)))
    eng = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=1 << 14)
    for bad in (B.BenchConfig(doc_grid=[64], reps=0), B.BenchConfig(doc_grid=[64], query_tokens=0)):
        with pytest.raises(T.DomainError):
            B.run_bench(eng, bad)
    config = B.BenchConfig(doc_grid=[512, 1024, 2048, 4096], query_tokens=64, reps=3, seed=42)
    rows = B.run_bench(eng, config)
    assert len(rows) == 4 * 2 * 3
    oc = O.qwen_layers(2)
    for r in rows:
        n = r.doc_tokens + r.query_tokens
        want = O.Port.flops_total(oc, r.query_tokens, n) if r.path == "turbo-reordered" else O.Port.flops_total(oc, n, n)
        assert r.measured_flops == want
    summary = B.summarize(rows)
    speedups = [s.speedup for s in summary]
    assert speedups == sorted(speedups), f"speedup not monotone over the grid: {speedups}"
    assert summary[-1].doc_tokens == 4096 and summary[-1].turbo_median_ms * 3.0 <= summary[-1].naive_median_ms
    eng.close()


def test_flops_model_matches_reference_compare():
    from paper_2410_07590_b200 import pipeline_api as P
    cfg = T.ModelConfig.qwen2_7b_like()
    cmp = P.compare(cfg, 8192, 128)
    assert cmp.naive.total == O.Port.flops_total(O.QWEN2_7B, 8320, 8320)
    assert cmp.turbo.total == O.Port.flops_total(O.QWEN2_7B, 128, 8320)
    assert abs(cmp.reduction_percent - 98.4615) < 1e-3  # proj/README.md:137-138
    with pytest.raises(T.DomainError):
        P.flops(cfg, 8, 4)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_answer_matches_reference_engine(tmp_path, mode):
    """Engine::answer end to end (retrieval on the GPU index, KV injection or full concat, greedy decode) on the
    toy model in f32: same retrieved chunk ids, same answer tokens, same prefill / modeled / decode FLOP counts."""
    from paper_2410_07590_b200 import pipeline_api as P
    if not O.Ref.available():
        pytest.skip("reference sources absent (GPU box)")
    pays = [O.random_text_tokens(3000 + i, 126) for i in range(6)]
    eng = T.Engine(T.ModelConfig.toy(), 42, dtype="f32", store_capacity_tokens=4096)
    eng.ingest_chunks(pays)
    ref = O.RefEngine(O.TOY, 42, str(tmp_path / "store"))
    try:
        for p in pays:
            ref.ingest(p)
        question = "which document mentions the river"
        want = ref.answer(question, 3, mode, 8)
        got = P.answer(eng, question, 3, P.PathMode(mode), 8)
        assert got.retrieved == want["retrieved"]
        assert got.tokens == want["tokens"]
        for key in ("prefill_flops", "modeled_prefill_flops", "decode_flops", "context_tokens", "query_tokens"):
            assert getattr(got, key) == want[key], key
        assert got.prefill_flops == got.modeled_prefill_flops
        assert got.text == P.decode(want["tokens"]) and got.ttft_ms > 0
    finally:
        ref.close()
        eng.close()
    with pytest.raises(T.DomainError):
        P.answer(T.Engine(T.ModelConfig.toy(), 42, dtype="f32", store_capacity_tokens=1024), "", 1,
                 P.PathMode.TurboReordered, 1)


CHUNK_TEXTS = [
    b"", b"x", b"short text", b"the quick brown fox jumps over the lazy dog " * 30,
    b"a" * 100, b"word\tword\nword\rword\fword\vword  " * 20, bytes(range(32, 127)) * 9,
]


@pytest.mark.parametrize("target", [8, 12, 32, 48, 100, 256])
def test_chunk_document_matches_reference(target):
    from paper_2410_07590_b200 import pipeline_api as P
    for text in CHUNK_TEXTS:
        chunks = P.chunk_document(text.decode("latin-1") if max(text, default=0) < 128 else text.decode(), target)
        assert b"".join(bytes(c.astype(np.uint8)) for c in chunks) == text  # lossless
        assert all(0 < len(c) <= target for c in chunks)
        if O.Ref.available():
            assert [len(c) for c in chunks] == O.ref_chunk_lengths(text, target)
    with pytest.raises(T.DomainError):
        P.chunk_document("x", 7)


def _unit_config():
    return T.ModelConfig(layer_num=1, head_num=1, kv_head_num=1, head_size=2, hidden_size=2, intermediate_size=1,
                         vocab_size=1)


def test_costmodel_reference_cases():
    """proj/tests/test_costmodel.cpp, case by case."""
    from paper_2410_07590_b200 import pipeline_api as P
    r = P.flops(_unit_config(), 1, 1, 1)
    assert (r.c_qkv, r.c_attn, r.c_o, r.c_mlp, r.total) == (24, 4, 8, 12, 48)
    r10 = P.flops(_unit_config(), 1, 10, 1)
    assert r10.c_attn == 40 and (r10.c_qkv, r10.c_o, r10.c_mlp) == (r.c_qkv, r.c_o, r.c_mlp)
    q = T.ModelConfig.qwen2_7b_like()
    base = P.flops(q, 128, 8320, 1)
    assert P.flops(q, 128, 8320, 2).total == 2 * base.total and P.flops(q, 128, 8320, 4).total == 4 * base.total
    assert P.flops(q, 256, 8320, 1).total == 2 * base.total
    half = T.ModelConfig(**{**vars(q), "layer_num": q.layer_num // 2})
    assert 2 * P.flops(half, 128, 8320, 1).total == base.total
    cmp = P.compare(q, 8192, 128, 1)
    assert abs(cmp.naive.tflops() - 136.36) <= 0.15 * 136.36 and abs(cmp.reduction_percent - 98.46) < 0.5
    assert (cmp.turbo.n_input, cmp.turbo.n_context, cmp.naive.n_input) == (128, 8320, 8320)
    none = P.compare(q, 0, 128, 1)
    assert none.reduction_percent == 0.0 and none.naive.total == none.turbo.total
    reds = [P.compare(q, c, 128, 1).reduction_percent for c in (512, 2048, 8192, 32768)]
    assert reds == sorted(reds) and reds[-1] < 100.0
    firsts = [P.compare(T.ModelConfig(**{**vars(q), "layer_num": n}), 8192, 128, 1).reduction_percent for n in (1, 4, 28)]
    assert max(firsts) - min(firsts) <= 1e-12 * firsts[0]
    toy = T.ModelConfig.toy()
    for args in ((0, 1, 1), (1, 0, 1), (1, 1, 0), (5, 4, 1)):
        with pytest.raises(T.DomainError):
            P.flops(toy, *args)
    for args in ((-1, 8, 1), (8, 0, 1)):
        with pytest.raises(T.DomainError):
            P.compare(toy, *args)
    with pytest.raises(T.ConfigError):
        P.flops(T.ModelConfig(**{**vars(toy), "head_size": 0}), 1, 1, 1)
    flat = P.flops(toy, 100, 100, 1)
    ramped = P.flops_attention_ramped(toy, 100, 0)
    assert ramped < toy.layer_num * 100 * flat.c_attn
    assert ramped == toy.layer_num * 2 * toy.head_num * toy.head_size * (100 * 101 // 2)


def test_path_mode_names_round_trip():
    """proj/tests/test_pipeline.cpp:56-64"""
    from paper_2410_07590_b200 import pipeline_api as P
    for m in P.PathMode:
        assert P.path_mode_from_string(P.to_string(m)) == m
    with pytest.raises(T.ConfigError):
        P.path_mode_from_string("fast")
    assert P.to_string(T.PositionMode.Composite) == "composite" and P.to_string(T.PositionMode.Reordered) == "reordered"


def test_flops_report_schema():
    """docs/formats.md "JSON reports" (flops): keys, rows per batch, totals from the cost model."""
    from paper_2410_07590_b200 import pipeline_api as P
    rep = P.flops_report("qwen2-7b", 8192, 128)
    assert rep["schema"] == "turbokv-report/1" and rep["command"] == "flops"
    assert set(rep) == {"schema", "command", "preset", "chunk_tokens", "query_tokens", "config", "rows"}
    assert [r["batch"] for r in rep["rows"]] == [1, 2, 4, 6, 8]
    r1 = rep["rows"][0]
    assert set(r1) == {"batch", "naive_total", "turbo_total", "naive_tflops", "turbo_tflops", "reduction_percent"}
    assert r1["naive_total"] == O.Port.flops_total(O.QWEN2_7B, 8320, 8320)
    assert 100.0 < r1["naive_tflops"] < 160.0  # proj/tests/test_cli.cpp flops --json bounds
    with pytest.raises(T.ConfigError):
        P.flops_report("qwen2-7b", 0, 128)


@pytest.mark.gpu
def test_ask_report_schema():
    from paper_2410_07590_b200 import pipeline_api as P
    eng = T.Engine(T.ModelConfig.toy(), 42, dtype="f32", store_capacity_tokens=4096)
    ref = P.ask_report(eng, "anything?", 2, "turbo-reordered", 4)
    assert ref == {"schema": "turbokv-report/1", "command": "ask", "refused": True, "reason": "no documents ingested"}
    P.ingest(eng, [P.Document("d", "canal locks hold water between gates while boats rise or fall")], 24)
    rep = P.ask_report(eng, "how do locks work?", 2, "naive-independent", 4)
    assert {"schema", "command", "refused", "mode", "question", "answer_text", "answer_tokens", "retrieved",
            "timings_ms", "flops", "context_tokens", "query_tokens", "seed", "config"} == set(rep)
    assert rep["refused"] is False and all(len(h) == 16 for h in rep["retrieved"])
    assert rep["flops"]["prefill_measured"] == rep["flops"]["prefill_modeled"]
    assert set(rep["timings_ms"]) == {"retrieval", "cache_load", "ttft", "decode"}
    eng.close()


def test_verify_helpers_follow_reference(golden):
    """`turbokv verify` case generation (tools/turbokv_main.cpp:167-174, 349-375): SplitMix64::at per case seed (the
    reference's own golden streams), random_text over 'a'..'z' + space, next_signed in [-1, 1), and the RoPE
    relative score's shift invariance at 1e-9."""
    from paper_2410_07590_b200 import pipeline_api as P
    from paper_2410_07590_b200.bench_api import SplitMix64
    meta, _ = golden
    for seed, outs in meta["splitmix"].items():
        for i, h in enumerate(outs):
            assert P._splitmix_at(int(seed), i) == int(h, 16)
    rng = SplitMix64(7)
    txt = P._random_text(rng, 500)
    assert len(txt) == 500 and set(txt) <= set("abcdefghijklmnopqrstuvwxyz ")
    xs = [P._next_signed(rng) for _ in range(1000)]
    assert -1.0 <= min(xs) and max(xs) < 1.0
    q, k = [P._next_signed(rng) for _ in range(64)], [P._next_signed(rng) for _ in range(64)]
    assert abs(P._rope_relative_score(q, k, 10, 300, 1e4) - P._rope_relative_score(q, k, 1010, 1300, 1e4)) < 1e-9
    assert abs(P._rope_relative_score(q, k, 10, 300, 1e4) - P._rope_relative_score(q, k, 10, 301, 1e4)) > 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_verify_properties_hold_and_fault_is_caught(dtype, tmp_path):
    """`turbokv verify` (tools/turbokv_main.cpp:586-606) over the engine: every property holds (equivalence with
    identical decodes and a composite-defect witness, RoPE shift invariance, KV round trip and its error paths,
    incremental == one-shot, single-chunk degeneracy); with --inject-fault the f32 engine's equivalence check fails
    and prints the reproduction line, as in the (f64) reference."""
    from paper_2410_07590_b200 import pipeline_api as P
    eng = T.Engine(T.ModelConfig.toy(), 42, dtype=dtype, store_capacity_tokens=1 << 16)
    rc, lines = P.verify(eng, P.VerifyOpts(cases=12, rope_cases=200), str(tmp_path))
    assert rc == 0, lines
    assert lines[0] == "ok equivalence (12 cases)" and lines[1].startswith("ok composite defect witness")
    assert lines[-1] == "all properties hold" and len(lines) == 7
    if dtype == "bf16":  # the fault moves toy logits by less than the bf16 bound: a precision (f32 / f64) check
        eng.close()
        return
    rc, lines = P.verify(eng, P.VerifyOpts(cases=3, inject_fault=True), str(tmp_path))
    assert rc == 1 and lines[0].startswith("FAIL equivalence: logits diff")
    assert lines[1].startswith("REPRO: turbokv verify --case-seed ") and lines[1].endswith(" --cases 1 --inject-fault")
    eng.close()


@pytest.mark.gpu
def test_ingest_report_schema():
    """`turbokv ingest --json` (tools/turbokv_main.cpp:218-231): keys and counts; re-ingesting adds no new chunks."""
    from paper_2410_07590_b200 import pipeline_api as P
    eng = T.Engine(T.ModelConfig.toy(), 42, dtype="f32", store_capacity_tokens=4096)
    docs = [P.Document("a", "canal locks hold water between gates while boats rise or fall"),
            P.Document("b", "a lighthouse keeper trims the wick every night")]
    rep = P.ingest_report(eng, docs, 24, "store", "toy", "f32")
    assert set(rep) == {"schema", "command", "store", "documents", "chunks", "new_chunks", "bytes_written",
                        "indexed_chunks", "seed", "preset", "dtype", "config"}
    assert rep["command"] == "ingest" and rep["documents"] == 2 and rep["chunks"] == rep["new_chunks"] > 0
    assert rep["indexed_chunks"] == rep["chunks"]
    again = P.ingest_report(eng, docs, 24, "store", "toy", "f32")
    assert again["new_chunks"] == 0 and again["chunks"] == rep["chunks"]
    eng.close()
