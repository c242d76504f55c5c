"""The reference's pipeline / model behaviour cases (proj/tests/test_pipeline.cpp:74-99, 276-309 and
proj/tests/test_model.cpp:196-247) on the B200 engine through the caller mirrors (pipeline_api.py)."""
import numpy as np
import pytest

from paper_2410_07590_b200 import pipeline_api as P
from paper_2410_07590_b200 import turbokv as T

pytestmark = pytest.mark.gpu

DOCS = [
    P.Document("locks", "A pound lock holds water between two gates. Boats enter, the chamber fills or drains, and "
                        "the far gate opens once the levels match. Paddles in the gates let the water through."),
    P.Document("tides", "Tides rise and fall twice a day because the moon and the sun pull on the oceans. Spring "
                        "tides are the largest; neap tides are the smallest."),
    P.Document("bread", "Bread rises when yeast turns sugar into gas. Kneading builds gluten that traps the gas; "
                        "baking sets the crumb and browns the crust."),
]


def toy_engine(cap=1 << 14):
    return T.Engine(T.ModelConfig.toy(), 42, dtype="f32", store_capacity_tokens=cap)


def test_ingest_is_lossless_and_idempotent():
    eng = toy_engine()
    first = P.ingest(eng, DOCS, 40)
    assert first.chunks > 3 and first.new_chunks == first.chunks and first.bytes_written > 0
    assert eng.index_size() == first.chunks
    payload_bytes = sum(len(eng.chunk_framed_tokens(i)) - 2 for i in eng._framed)
    assert payload_bytes == sum(len(d.text.encode()) for d in DOCS)
    again = P.ingest(eng, DOCS, 40)
    assert again.chunks == first.chunks and again.new_chunks == 0 and again.bytes_written == 0
    assert eng.index_size() == first.chunks
    eng.close()


def test_answer_identical_across_turbo_and_naive():
    eng = toy_engine()
    P.ingest(eng, DOCS, 48)
    q = "how does a pound lock work?"
    turbo = P.answer(eng, q, 3, P.PathMode.TurboReordered, 16)
    naive = P.answer(eng, q, 3, P.PathMode.NaiveIndependent, 16)
    assert turbo.retrieved == naive.retrieved and turbo.tokens == naive.tokens and turbo.text == naive.text
    assert (turbo.context_tokens, turbo.query_tokens) == (naive.context_tokens, naive.query_tokens)
    assert turbo.prefill_flops == turbo.modeled_prefill_flops and naive.prefill_flops == naive.modeled_prefill_flops
    assert turbo.prefill_flops < naive.prefill_flops and turbo.decode_flops > 0
    eng.close()


def test_answer_refuses_without_context_and_rejects_empty_questions():
    eng = toy_engine()
    with pytest.raises(T.NoContextError):
        P.answer(eng, "anything?", 2, P.PathMode.TurboReordered, 4)
    eng.ingest_chunk_payload("d", P.encode("now there is context"))
    with pytest.raises(T.DomainError):
        P.answer(eng, "", 2, P.PathMode.TurboReordered, 4)
    r = P.answer(eng, "what is here?", 50, P.PathMode.TurboReordered, 4)  # k beyond the index: everything
    assert len(r.retrieved) == 1
    eng.close()


def test_greedy_decode_deterministic_and_grows_context():
    eng = toy_engine()
    prompt = P.encode("the sea was calm")
    outs = []
    for _ in range(2):
        with eng.assemble([], T.PositionMode.Reordered) as ctx:
            eng.prefill_query(ctx, prompt)
            out = eng.greedy_decode(ctx, 12)
            assert ctx.total_tokens() == len(prompt) + len(out)
            assert ctx.next_position == ctx.total_tokens() and ctx.positions[-1] == ctx.total_tokens() - 1
            outs.append(out)
    assert outs[0] == outs[1]
    eng.close()


def test_decode_edge_cases():
    eng = toy_engine()
    prompt = P.encode("abc")
    with eng.assemble([], T.PositionMode.Reordered) as ctx:
        eng.prefill_query(ctx, prompt)
        assert eng.greedy_decode(ctx, 0) == [] and ctx.total_tokens() == 3  # max_new = 0 emits nothing
        with pytest.raises(T.DomainError):
            eng.greedy_decode(ctx, -1)
    with eng.assemble([], T.PositionMode.Reordered) as ctx:  # never prefilled: no logits to decode from
        with pytest.raises(T.DomainError):
            eng.greedy_decode(ctx, 4)
    eng.close()


def test_engine_requires_tokenizer_sized_vocabulary():
    """proj/tests/test_pipeline.cpp:66-72: structurally valid, too small for the 259-id tokenizer."""
    cfg = T.ModelConfig(**{**vars(T.ModelConfig.toy()), "vocab_size": 128})
    cfg.validate()
    with pytest.raises(T.ConfigError):
        T.Engine(cfg, 1, dtype="f32", store_capacity_tokens=1024)


def test_store_ids_sorted_and_ingest_is_a_noop_for_known_ids():
    """proj/tests/test_kvstore.cpp:89-110: storing the same id twice is a no-op; ids come back sorted."""
    eng = toy_engine()
    pays = [P.encode(f"chunk number {i} " * (3 + i)) for i in (5, 1, 4, 2, 3)]
    ids = eng.ingest_chunks(pays)
    assert eng.store_ids() == sorted(ids)
    st = T.IngestStats()
    assert eng.ingest_chunks(pays[:2], st) == ids[:2] and st.new_chunks == 0 and st.bytes_written == 0
    assert eng.store_ids() == sorted(ids)
    eng.store_evict(ids[0])
    assert eng.store_ids() == sorted(ids[1:])
    eng.close()


def test_tier_rebalance_promotes_hot_chunks_and_keeps_kv_bitwise():
    """tkv_store_rebalance (the C4 two-tier policy): chunks retrieved often from the pinned host tier move into HBM,
    the coldest HBM chunks move out, and a request over moved chunks gives bitwise the logits it gave before."""
    import oracle as O
    eng = T.Engine(T.ModelConfig.toy(), 42, dtype="bf16", store_capacity_tokens=4 * 64, host_spill_tokens=8 * 64)
    try:
        pays = [O.random_text_tokens(4400 + i, 62) for i in range(8)]
        ids = eng.ingest_chunks(pays)
        assert [eng.store_chunk_tier(i) for i in ids] == [0] * 4 + [1] * 4  # HBM fills first
        hot = ids[5:8]
        q = O.random_text_tokens(77, 12)
        with eng.assemble(hot, T.PositionMode.Reordered) as ctx:
            before = eng.prefill_query(ctx, q).copy()
        for _ in range(3):
            eng.assemble(hot, T.PositionMode.Reordered).close()
        up, down = eng.store_rebalance()
        assert up == 3 and down == 3
        assert all(eng.store_chunk_tier(i) == 0 for i in hot)
        assert sum(eng.store_chunk_tier(i) == 1 for i in ids) == 4
        with eng.assemble(hot, T.PositionMode.Reordered) as ctx:
            after = eng.prefill_query(ctx, q).copy()
        assert np.array_equal(before, after)
        for i in ids:  # every chunk still reads back (demoted ones from the host tier)
            assert np.isfinite(eng.store_read(i, 0, "k")).all()
        assert eng.store_rebalance() == (0, 0)  # nothing hotter left outside HBM
    finally:
        eng.close()
