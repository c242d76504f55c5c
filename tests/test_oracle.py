"""CPU: the oracle restatement (oracle/tkv_oracle.c) pinned against the reference's golden
vectors (tests/golden/, generated from the reference itself by make_golden.py) and, where
/root/reference is present, against the reference library built in place (oracle/_ref)."""
import numpy as np
import pytest

import oracle as O


def cfg_of(meta):
    return O.Cfg(**meta["config"])


def test_splitmix_canonical_vectors(golden):
    meta, _ = golden
    # proj/docs/formats.md:45-52
    assert meta["splitmix"]["0"] == ["e220a8397b1dcdaf", "6e789e6aa1b965f4", "06c45d188009454f"]
    assert [int(x, 16) for x in meta["splitmix"]["1234567"]] == [
        6457827717110365317, 3203168211198807973, 9817491932198370423]
    for seed, outs in meta["splitmix"].items():
        for i, h in enumerate(outs):
            assert O.Port.lib().tko_splitmix_at(int(seed), i) == int(h, 16)
            assert O.splitmix_at(int(seed), i) == int(h, 16)
    u = (O.splitmix_at(42, 0) >> 11) * 2.0 ** -53
    assert u == 0.74156487877182331


def test_toy_weight_identity(golden):
    meta, _ = golden
    g = meta["toy_identity"]
    assert g["checksum42"] == "783fe06586f74dc9" and g["fingerprint42"] == "8dd32810bd252fd1"
    p = O.Port(O.TOY, 42)
    assert p.checksum() == int(g["checksum42"], 16)
    assert p.fingerprint() == int(g["fingerprint42"], 16)
    assert p.weight(0, 0)[0, 0] == g["emb00"] == 0.060391219692955828
    assert O.Port(O.TOY, 7).checksum() == int(g["checksum7"], 16)
    # draw order: wq(0,0) continues right after the embedding (proj/tests/test_model.cpp:83-91)
    p9 = O.Port(O.TOY, 9)
    n = O.TOY.vocab_size * O.TOY.hidden_size
    u = (O.splitmix_at(9, n) >> 11) * 2.0 ** -53
    assert p9.weight(0, 1)[0, 0] == (2.0 * u - 1.0) * 0.125


def test_positions_345(golden):
    meta, _ = golden
    for reordered, tag in ((True, "reordered"), (False, "composite")):
        pos, nxt = O.Port.assemble_positions([3, 4, 5], reordered)
        assert pos.tolist() == meta[f"positions_345.{tag}"]["positions"]
        assert nxt == meta[f"positions_345.{tag}"]["next"]


def dense(lo, hi, cols):
    j = np.arange(cols)[None, :]
    return ((j >= lo[:, None]) & (j <= hi[:, None])).astype(np.uint8)


def test_mask_rows_match_reference_masks(golden):
    _, A = golden
    for independent, tag in ((False, "causal"), (True, "independent")):
        lo, hi = O.Port.mask_rows([3, 4, 5, 2], independent)
        assert (dense(lo, hi, 14) == A[f"mask.3452.{tag}"]).all()
    lo, hi = O.Port.causal_rows(5, 7)
    assert (dense(lo, hi, 12) == A["mask.causal_rows_5_7"]).all()


@pytest.mark.parametrize("name", ["c1", "ragged"])
def test_paths_bit_exact_vs_golden(golden, name):
    meta, A = golden
    m = meta[name]
    cfg = cfg_of(m)
    p = O.Port(cfg, m["seed"])
    assert f"{p.fingerprint():016x}" == m["fingerprint"]
    offs = A[f"{name}.payload_offsets"]
    pays = [A[f"{name}.payloads"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
    framed = [O.frame(x) for x in pays]
    assert [f"{p.chunk_id(f):016x}" for f in framed] == m["ids"]
    q = A[f"{name}.query"]
    for reordered, tag in ((True, "reordered"), (False, "composite")):
        k, v, pos, nxt = p.assemble(framed, reordered)
        assert (pos == A[f"{name}.{tag}.positions"]).all() and nxt == m[f"{tag}.next_position"]
        logits = p.prefill_query(k, v, pos, nxt, q)
        assert np.array_equal(logits, A[f"{name}.turbo_{tag}.logits"])
        if reordered:
            for key in A:
                if key.startswith(f"{name}.k") and not key.startswith(f"{name}.krot"):
                    layer = int(key[len(name) + 2:])
                    assert np.array_equal(k[layer], A[key])
                    assert np.array_equal(v[layer], A[f"{name}.v{layer}"])
                    rot = O.Port.rope(k[layer], pos, cfg.head_size, cfg.rope_base)
                    assert np.array_equal(rot, A[f"{name}.krot{layer}"])
    for independent, tag in ((False, "causal"), (True, "independent")):
        assert np.array_equal(p.naive_prefill(framed, q, independent), A[f"{name}.naive_{tag}.logits"])
    # TurboRAG equivalence (proj/tests/test_pipeline.cpp:182-208): turbo == naive-independent <= 1e-10
    assert np.abs(A[f"{name}.turbo_reordered.logits"] - A[f"{name}.naive_independent.logits"]).max() <= 1e-10
    # composite defect (test_pipeline.cpp:210-234) is visible on the multi-chunk C1 case
    if name == "c1":
        assert np.abs(A["c1.turbo_composite.logits"] - A["c1.naive_independent.logits"]).max() > 1e-3


@pytest.mark.slow
def test_qwen_dims_one_layer_vs_golden(golden):
    meta, A = golden
    m = meta["qwen1"]
    p = O.Port(cfg_of(m), m["seed"])
    offs = A["qwen1.payload_offsets"]
    framed = [O.frame(A["qwen1.payloads"][offs[i]:offs[i + 1]]) for i in range(len(offs) - 1)]
    k, v, pos, nxt = p.assemble(framed, True)
    assert np.array_equal(k[0], A["qwen1.k0"])
    logits = p.prefill_query(k, v, pos, nxt, A["qwen1.query"])
    assert np.array_equal(logits, A["qwen1.turbo_reordered.logits"])


def test_flops_model_matches_reference_counter(golden):
    meta, _ = golden
    m = meta["c1"]
    cfg = cfg_of(m)
    # FlopCounter::add_forward charges n_ctx = past + new (costmodel.cpp:77-83)
    assert sum(m["turbo_reordered.flops"]) == O.Port.flops_total(cfg, 32, 512 + 32)
    # Appendix C comparison, batch 1, 8192 + 128 on Qwen2-7B: 98.4615 % (proj/README.md:137-138)
    naive = O.Port.flops_total(O.QWEN2_7B, 8320, 8320)
    turbo = O.Port.flops_total(O.QWEN2_7B, 128, 8320)
    assert abs(100 * (1 - turbo / naive) - 98.4615) < 1e-3


@pytest.mark.skipif(not O.Ref.available(), reason="reference sources absent (GPU box)")
def test_restatement_equals_reference_random_grid(tmp_path):
    """Acceptance-style grid (proj/tests/acceptance_main.cpp:80-139), restatement vs reference."""
    rng = np.random.default_rng(5)
    for seed in (42, 7):
        eng = O.RefEngine(O.TOY, seed, str(tmp_path / f"s{seed}"))
        p = O.Port(O.TOY, seed)
        for case in range(4):
            lens = rng.integers(1, 65, size=int(rng.integers(1, 9)))
            pays = [O.random_text_tokens(seed * 100 + case * 10 + i, int(n)) for i, n in enumerate(lens)]
            ids = [eng.ingest(x) for x in pays]
            q = O.random_text_tokens(case + 1, int(rng.integers(1, 33)))
            ctx = eng.assemble(ids, True)
            ref_logits, _ = ctx.prefill_query(q)
            framed = [O.frame(x) for x in pays]
            k, v, pos, nxt = p.assemble(framed, True)
            assert np.array_equal(p.prefill_query(k, v, pos, nxt, q), ref_logits)


def test_retrieval_restatement_matches_reference():
    """embed (retrieval.cpp:64-88) and top_k (retrieval.cpp:117-133): the C restatement against the reference
    itself, bit for bit, including cosine ties broken by ascending chunk id and the cancelled-counts edge case."""
    rng = np.random.default_rng(5)
    docs = [O.random_text_tokens(100 + i, int(rng.integers(1, 300))) for i in range(60)]
    docs += [np.array([97, 98], np.int32), np.array([97], np.int32)]
    docs += [docs[3].copy(), docs[7].copy()]  # duplicates: identical cosines, tie-break by id
    emb = np.stack([O.Port.embed(d) for d in docs])
    for d, e in zip(docs, emb):
        assert np.array_equal(e, O.Ref.embed(d))
        assert abs(np.linalg.norm(e) - 1.0) < 1e-12
    ids = rng.permutation(np.arange(1, len(docs) + 1, dtype=np.uint64) * 0x9E3779B97F4A7C15)
    for qseed in range(5):
        q = O.Port.embed(O.random_text_tokens(7000 + qseed, 50))
        for k in (1, 5, 16, 200):
            got, scores = O.Port.top_k(emb, ids, q, k)
            assert np.array_equal(got, O.Ref.top_k(emb, ids, q, k))
            assert np.all(np.diff(scores) <= 0)
    with pytest.raises(O.OracleError):
        O.Port.top_k(emb, ids, q, 0)


def test_streamed_identity_equals_reference(golden):
    """The streamed weights_checksum (no materialised weights; used for the full-size identities in
    tests/golden/identity_full.json) equals the reference's own checksum at every size it can hold here."""
    meta, _ = golden
    g = meta["toy_identity"]
    assert O.Port.stream_identity(O.TOY, 42) == (int(g["checksum42"], 16), int(g["fingerprint42"], 16))
    assert O.Port.stream_identity(O.TOY, 7)[0] == int(g["checksum7"], 16)
    q1 = meta["qwen1"]
    assert O.Port.stream_identity(cfg_of(q1), q1["seed"])[1] == int(q1["fingerprint"], 16)
    if O.Ref.available():
        for cfg, seed in ((O.Cfg(2, 4, 2, 16, 64, 96), 5), (O.Cfg(1, 8, 8, 32, 256, 512, 300, 5e5, 1e-5), 11)):
            assert O.Port.stream_identity(cfg, seed) == O.Ref.identity(cfg, seed)[:2]


def test_large_golden_ids_follow_the_reference_identity():
    """golden_large chunk ids are FNV(fingerprint, framed tokens) under the case's reference fingerprint."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_large.json")
    meta = json.load(open(path))
    A = np.load(path.replace(".json", ".npz"))
    for name, m in meta.items():
        fp = int(m["fingerprint"], 16)
        offs = A[f"{name}.payload_offsets"]
        pays = [A[f"{name}.payloads"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
        for p, cid in zip(pays, m["ids"]):
            f = O.frame(p)
            assert O.Port.lib().tko_chunk_content_id(fp, f.ctypes.data_as(O.I32P), len(f)) == int(cid, 16)
