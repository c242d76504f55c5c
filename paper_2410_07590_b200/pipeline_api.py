"""Engine::answer (src/pipeline.cpp:247-308) and the Appendix-C cost model (src/costmodel.cpp:11-83) over the B200
engine: the reference's top-level caller of the hot path (retrieval -> KV injection or full-concat prefill ->
first-token logits -> greedy decode), with the same result fields (include/turbokv/pipeline.hpp:42-55).

Retrieval runs on the GPU index (cosine top-k, ranking bit-identical to RetrievalIndex::top_k), the turbo
window covers assemble (KV gather + RoPE) and the query prefill, the naive window the full-concat prefill with
the chunk tokens in hand; decode FLOPs are counted per generated token as forward_tokens' FlopCounter does
(add_forward with one new token over the grown context).
"""
from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field

import numpy as np

from . import turbokv as T

PREAMBLE = ("Answer the question using only the documents provided. "
            "If the documents do not contain the answer, refuse to answer.\n"
            "Question: ")  # pipeline.cpp:20-23
DOC_START, DOC_END, EOS = 256, 257, 258


class PathMode(enum.IntEnum):
    """pipeline.hpp:25"""
    TurboReordered = 0
    TurboComposite = 1
    NaiveCausal = 2
    NaiveIndependent = 3


_PATH_NAMES = {PathMode.TurboReordered: "turbo-reordered", PathMode.TurboComposite: "turbo-composite",
               PathMode.NaiveCausal: "naive-causal", PathMode.NaiveIndependent: "naive-independent"}


def to_string(mode) -> str:
    """pipeline.cpp:31-43 (PathMode and PositionMode names)."""
    if isinstance(mode, PathMode):
        return _PATH_NAMES[mode]
    return "composite" if mode == T.PositionMode.Composite else "reordered"


def path_mode_from_string(name: str) -> PathMode:
    """pipeline.cpp:45-53"""
    for m, n in _PATH_NAMES.items():
        if n == name:
            return m
    raise T.ConfigError(f"unknown mode '{name}' (expected turbo-reordered, turbo-composite, naive-causal, "
                        "or naive-independent)")


@dataclass
class FlopsReport:
    """costmodel.hpp FlopsReport"""
    c_qkv: int
    c_attn: int
    c_o: int
    c_mlp: int
    n_input: int
    n_context: int
    batch: int
    total: int

    def tflops(self) -> float:
        return self.total / 1e12


def _validated(config: T.ModelConfig) -> T.ModelConfig:
    config.validate()  # ModelConfig::validate (config.cpp:9-40): ConfigError
    return config


def flops(config: T.ModelConfig, n_input: int, n_context: int, batch: int = 1) -> FlopsReport:
    """costmodel.cpp:28-46 (Appendix C): total = batch * n_input * L * (c_qkv + c_attn(n_context) + c_o + c_mlp)."""
    _validated(config)
    if n_input < 1 or n_context < 1 or batch < 1:
        raise T.DomainError("flops: n_input, n_context and batch must be >= 1")
    if n_context < n_input:
        raise T.DomainError("flops: n_context < n_input")
    c = config
    qkv = 2 * c.hidden_size * (c.head_num + 2 * c.kv_head_num) * c.head_size
    attn = 2 * c.head_num * c.head_size * n_context
    o = 2 * c.hidden_size * c.hidden_size
    mlp = 2 * 3 * c.hidden_size * c.intermediate_size
    return FlopsReport(qkv, attn, o, mlp, n_input, n_context, batch, batch * n_input * c.layer_num * (qkv + attn + o + mlp))


def flops_attention_ramped(config: T.ModelConfig, n_input: int, past: int) -> int:
    """costmodel.cpp:65-75: attention charged per token over the context it actually sees (token t: past + t + 1)."""
    _validated(config)
    if n_input < 1 or past < 0:
        raise T.DomainError("flops_attention_ramped: bad counts")
    per = 2 * config.head_num * config.head_size
    return config.layer_num * per * (n_input * past + n_input * (n_input + 1) // 2)


@dataclass
class FlopsComparison:
    naive: FlopsReport
    turbo: FlopsReport
    reduction_percent: float


def compare(config: T.ModelConfig, chunk_tokens: int, query_tokens: int, batch: int = 1) -> FlopsComparison:
    """costmodel.cpp:48-62"""
    if chunk_tokens < 0 or query_tokens < 1:
        raise T.DomainError("compare: need chunk_tokens >= 0 and query_tokens >= 1")
    total = chunk_tokens + query_tokens
    naive, turbo = flops(config, total, total, batch), flops(config, query_tokens, total, batch)
    return FlopsComparison(naive, turbo, 100.0 * (1.0 - turbo.total / naive.total))


@dataclass
class Document:
    """pipeline.hpp:31-34"""
    id: str
    text: str


_SPACE = frozenset(b" \t\n\r\f\v")  # retrieval.cpp:16-18


def chunk_document(text: str, target_len: int) -> list:
    """retrieval.cpp:32-58: byte windows of target_len, each ending after the window's last whitespace byte
    when it has one (the whitespace stays left, so concatenating the chunks gives the text back)."""
    if target_len < 8:
        raise T.DomainError("chunk_document: target_len must be >= 8")
    data = text.encode("utf-8")
    out, pos, n = [], 0, len(data)
    while pos < n:
        take = min(target_len, n - pos)
        if pos + take < n:
            for i in range(take, 0, -1):
                if data[pos + i - 1] in _SPACE:
                    take = i
                    break
        out.append(np.frombuffer(data[pos:pos + take], np.uint8).astype(np.int32))
        pos += take
    return out


def ingest(engine: T.Engine, docs, target_len: int) -> T.IngestStats:
    """Engine::ingest (pipeline.cpp:81-95): every document chunked and its chunks precomputed (one batched
    block-diagonal forward per document here); duplicates are counted but stored once."""
    stats = T.IngestStats()
    for doc in docs:
        payloads = chunk_document(doc.text, target_len)
        if not payloads:
            continue
        try:
            engine.ingest_chunks(payloads, stats)
        except T.Error as e:
            raise T.Error(f"ingest of document '{doc.id}' failed: {e}") from e
    return stats


@dataclass
class AnswerResult:
    """pipeline.hpp:42-55"""
    text: str = ""
    tokens: list = field(default_factory=list)
    retrieved: list = field(default_factory=list)
    retrieval_ms: float = 0.0
    cache_load_ms: float = 0.0  # inside ttft_ms for turbo paths
    ttft_ms: float = 0.0        # inputs ready -> first-token logits
    decode_ms: float = 0.0
    prefill_flops: int = 0
    modeled_prefill_flops: int = 0
    decode_flops: int = 0
    context_tokens: int = 0     # chunk tokens attended over
    query_tokens: int = 0


def encode(text: str) -> np.ndarray:
    return np.frombuffer(text.encode("utf-8"), np.uint8).astype(np.int32)


def decode(tokens) -> str:
    """tokenizer.cpp:17-34 (bytes -> text; invalid UTF-8 rendered with U+FFFD, as the JSON report does)."""
    out = bytearray()
    for t in tokens:
        if 0 <= t < 256:
            out.append(t)
        elif t == DOC_START:
            out += b"<|doc_start|>"
        elif t == DOC_END:
            out += b"<|doc_end|>"
        elif t == EOS:
            pass
        else:
            raise T.DomainError(f"decode: unknown token id {t}")
    return out.decode("utf-8", errors="replace")


def build_query_tokens(question: str) -> np.ndarray:
    """pipeline.cpp:243-245"""
    return encode(PREAMBLE + question + "\nAnswer:")


def answer(engine: T.Engine, question: str, k: int, mode: PathMode, max_new: int) -> AnswerResult:
    """pipeline.cpp:247-308"""
    if not question:
        raise T.DomainError("answer: empty question")
    if engine.index_size() == 0:
        raise T.NoContextError("nothing has been ingested; refusing to answer")
    cfg = engine.config
    r = AnswerResult()
    t0 = time.perf_counter()
    ids, _ = engine.top_k(encode(question), k)
    r.retrieved = [int(i) for i in ids]
    r.retrieval_ms = (time.perf_counter() - t0) * 1e3
    q = build_query_tokens(question)
    r.query_tokens = len(q)
    r.context_tokens = sum(engine.store_chunk_tokens(i) for i in r.retrieved)
    total = r.context_tokens + r.query_tokens
    counter = T.FlopCounter()
    if mode in (PathMode.TurboReordered, PathMode.TurboComposite):
        pos = T.PositionMode.Reordered if mode == PathMode.TurboReordered else T.PositionMode.Composite
        t0 = time.perf_counter()
        ctx = engine.assemble(r.retrieved, pos)
        r.cache_load_ms = (time.perf_counter() - t0) * 1e3
        engine.prefill_query(ctx, q, counter)
        r.ttft_ms = (time.perf_counter() - t0) * 1e3
        r.modeled_prefill_flops = flops(cfg, r.query_tokens, total).total
    else:
        mask = T.MaskMode.Causal if mode == PathMode.NaiveCausal else T.MaskMode.Independent
        chunks = [engine.chunk_framed_tokens(i) for i in r.retrieved]
        t0 = time.perf_counter()
        ctx = engine.naive_prefill(chunks, q, mask, counter)
        r.ttft_ms = (time.perf_counter() - t0) * 1e3
        r.modeled_prefill_flops = flops(cfg, total, total).total
    r.prefill_flops = counter.total()
    try:
        t0 = time.perf_counter()
        r.tokens = engine.greedy_decode(ctx, max_new)
        r.decode_ms = (time.perf_counter() - t0) * 1e3
    finally:
        ctx.close()
    # forward_tokens charges add_forward(1 new token, past + 1) per generated token (model.cpp:270, 274-303)
    r.decode_flops = sum(flops(cfg, 1, total + i + 1).total for i in range(len(r.tokens)))
    r.text = decode(r.tokens)
    return r


# ---- turbokv-report/1 (docs/formats.md "JSON reports"; tools/turbokv_main.cpp:83-93, 220-310, 615-660) ----
REPORT_SCHEMA = "turbokv-report/1"


def hex_id(chunk_id: int) -> str:
    return f"{chunk_id:016x}"


def config_json(c: T.ModelConfig) -> dict:
    return {"layer_num": c.layer_num, "head_num": c.head_num, "kv_head_num": c.kv_head_num,
            "head_size": c.head_size, "hidden_size": c.hidden_size, "intermediate_size": c.intermediate_size,
            "vocab_size": c.vocab_size, "rope_base": c.rope_base, "norm_eps": c.norm_eps}


def ask_report(engine: T.Engine, question: str, k: int, mode: str, max_new: int) -> dict:
    """`turbokv ask --json`: the answer report, or the refusal report when nothing has been ingested."""
    try:
        r = answer(engine, question, k, path_mode_from_string(mode), max_new)
    except T.NoContextError:
        return {"schema": REPORT_SCHEMA, "command": "ask", "refused": True, "reason": "no documents ingested"}
    return {"schema": REPORT_SCHEMA, "command": "ask", "refused": False, "mode": mode, "question": question,
            "answer_text": r.text, "answer_tokens": list(r.tokens), "retrieved": [hex_id(i) for i in r.retrieved],
            "timings_ms": {"retrieval": r.retrieval_ms, "cache_load": r.cache_load_ms, "ttft": r.ttft_ms,
                           "decode": r.decode_ms},
            "flops": {"prefill_measured": r.prefill_flops, "prefill_modeled": r.modeled_prefill_flops,
                      "decode_measured": r.decode_flops},
            "context_tokens": r.context_tokens, "query_tokens": r.query_tokens, "seed": engine.seed,
            "config": config_json(engine.config)}


def flops_report(preset: str, chunk_tokens: int, query_tokens: int, batches=(1, 2, 4, 6, 8)) -> dict:
    """`turbokv flops --json`: the Appendix-C comparison per batch size."""
    if chunk_tokens < 1:
        raise T.ConfigError("flops: --chunk-tokens must be >= 1")
    if query_tokens < 1:
        raise T.ConfigError("flops: --query-tokens must be >= 1")
    config = T.ModelConfig.preset(preset)
    rows = []
    for b in batches:
        cmp = compare(config, chunk_tokens, query_tokens, b)
        rows.append({"batch": b, "naive_total": cmp.naive.total, "turbo_total": cmp.turbo.total,
                     "naive_tflops": cmp.naive.tflops(), "turbo_tflops": cmp.turbo.tflops(),
                     "reduction_percent": cmp.reduction_percent})
    return {"schema": REPORT_SCHEMA, "command": "flops", "preset": preset, "chunk_tokens": chunk_tokens,
            "query_tokens": query_tokens, "config": config_json(config), "rows": rows}



def ingest_report(engine: T.Engine, docs, chunk_bytes: int, store: str, preset: str, dtype: str) -> dict:
    """`turbokv ingest --json` (tools/turbokv_main.cpp:200-231): chunk + ingest the documents, report the counts."""
    stats = ingest(engine, docs, chunk_bytes)
    return {"schema": REPORT_SCHEMA, "command": "ingest", "store": store, "documents": len(docs),
            "chunks": stats.chunks, "new_chunks": stats.new_chunks, "bytes_written": stats.bytes_written,
            "indexed_chunks": engine.index_size(), "seed": engine.seed, "preset": preset, "dtype": dtype,
            "config": config_json(engine.config)}


# ---- `turbokv verify` (tools/turbokv_main.cpp:334-606): the property checks, run on this engine ----

@dataclass
class VerifyOpts:
    """VerifyOpts (turbokv_main.cpp:334-343)."""
    seed: int = 42
    case_seed: int = 0    # nonzero: run exactly this case, once
    cases: int = 40
    rope_cases: int = 1000
    chunks: int = 0       # 0 = randomize per case
    chunk_len: int = 0    # payload bytes, 0 = randomize
    query_len: int = 0    # tokens, 0 = randomize
    inject_fault: bool = False


def _random_text(rng, n: int) -> str:
    """random_text (turbokv_main.cpp:167-174): 'a'..'z' and space."""
    out = []
    for _ in range(n):
        r = rng.next_below(27)
        out.append(" " if r == 26 else chr(ord("a") + r))
    return "".join(out)


def _max_abs_diff(a, b) -> float:
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max())


def _rope_relative_score(q, k, pos_q: int, pos_k: int, base: float) -> float:
    """rope_relative_score (src/rope.cpp:90-104): <R(pos_q) q, R(pos_k) k> with interleaved pairs (2m, 2m+1),
    theta_m = base^(-2m/d) (rope.cpp:21-22, 35-46), in f64 -- the definition the engine's RoPE table is built from."""
    d = len(q)
    theta = np.array([base ** (-(2.0 * m) / d) for m in range(d // 2)])

    def rot(x, t):
        c, s = np.cos(float(t) * theta), np.sin(float(t) * theta)
        x0, x1 = x[0::2], x[1::2]
        y = np.empty(d)
        y[0::2], y[1::2] = x0 * c - x1 * s, x0 * s + x1 * c
        return y

    return float(np.dot(rot(np.asarray(q), pos_q), rot(np.asarray(k), pos_k)))


def verify(engine: T.Engine, opts: VerifyOpts | None = None, tmp_dir: str | None = None):
    """cmd_verify (turbokv_main.cpp:586-606) over this engine: equivalence (turbo == naive-independent, identical
    greedy decodes, a composite-defect witness), RoPE shift invariance, KV round trip with its error paths,
    incremental == one-shot prefill and single-chunk degeneracy, with the reference's case generation
    (SplitMix64::at(seed, i) per case) and report lines. Returns (exit code, lines).

    Tolerances: the reference compares f64 paths at 1e-10; here the turbo and naive paths run different kernels in
    the engine's dtype, so differences are bounded relative to max|logit| (f32 1e-4, bf16 2e-2, the parity bars of
    DESIGN.md §4), greedy decodes must agree token for token in f32 (bf16: the first token), and the composite
    witness must exceed max(1e-3, 5 x that bound). --inject-fault corrupts the naive path's mask exactly as the
    reference hook does (the last query row loses column 0); at f32 equivalence then fails as in the f64 reference,
    while at bf16 the toy fault stays inside the bf16 bound (a precision check is an f32 / f64 tool)."""
    import os
    import struct
    import tempfile

    from .bench_api import SplitMix64, encode

    opts = opts or VerifyOpts()
    if opts.cases < 1:
        raise T.ConfigError("verify: --cases must be >= 1")
    cfg = engine.config
    f32 = engine.dtype == T.Dtype.F32
    rel = 1e-4 if f32 else 2e-2
    lines: list[str] = []

    def repro(case_seed: int):
        lines.append(f"REPRO: turbokv verify --case-seed {case_seed} --cases 1"
                     + (" --inject-fault" if opts.inject_fault else ""))

    def naive_ids(ids, query, mode):
        if opts.inject_fault:  # testing::mask_fault_hook: mask(rows - 1, 0) = -inf
            n = sum(engine.store_chunk_tokens(i) for i in ids) + len(query)
            engine.set_mask_rows([-1], [1], [n - 1])
        return engine.naive_prefill_ids(ids, query, mode)

    # -- equivalence (turbokv_main.cpp:349-421)
    witness, multichunk, max_cdiff = False, False, 0.0
    for i in range(opts.cases):
        case_seed = opts.case_seed if opts.case_seed else _splitmix_at(opts.seed, i)
        rng = SplitMix64(case_seed)
        n_chunks = opts.chunks if opts.chunks > 0 else 1 + rng.next_below(8)
        ids = []
        for _ in range(n_chunks):
            ln = opts.chunk_len if opts.chunk_len > 0 else 1 + rng.next_below(64)
            ids.append(engine.ingest_chunk_payload("verify", encode(_random_text(rng, ln))))
        qlen = opts.query_len if opts.query_len > 0 else 1 + rng.next_below(32)
        query = encode(_random_text(rng, qlen))
        with engine.assemble(ids, T.PositionMode.Reordered) as turbo:
            tl = engine.prefill_query(turbo, query)[0]
            with naive_ids(ids, query, T.MaskMode.Independent) as naive:
                nl = naive.last_logits
                scale = max(float(np.abs(nl).max()), 1e-30)
                diff = _max_abs_diff(tl, nl)
                if diff > rel * scale:
                    lines.append(f"FAIL equivalence: logits diff {diff:g} (chunks {n_chunks}, query {qlen})")
                    repro(case_seed)
                    return 1, lines
                td, nd = engine.greedy_decode(turbo, 16), engine.greedy_decode(naive, 16)
                if (td != nd) if f32 else (td[:1] != nd[:1]):
                    lines.append(f"FAIL equivalence: greedy decodes diverge (chunks {n_chunks}, query {qlen})")
                    repro(case_seed)
                    return 1, lines
                if n_chunks >= 2:
                    multichunk = True
                    with engine.assemble(ids, T.PositionMode.Composite) as comp:
                        cl = engine.prefill_query(comp, query)[0]
                    cdiff = _max_abs_diff(cl, nl)
                    max_cdiff = max(max_cdiff, cdiff)
                    if cdiff > max(1e-3, 5 * rel * scale):
                        witness = True
        if opts.case_seed:
            break
    lines.append(f"ok equivalence ({opts.cases} cases)")
    if multichunk:
        if not witness:
            lines.append(f"FAIL composite witness: no multi-chunk case exceeded 1e-3 (max diff {max_cdiff:g})")
            repro(opts.seed)
            return 1, lines
        lines.append(f"ok composite defect witness (max diff {max_cdiff:g})")

    # -- RoPE shift invariance (turbokv_main.cpp:424-452)
    rng = SplitMix64(opts.seed ^ 0x0051CE)
    worst = 0.0
    for _ in range(opts.rope_cases):
        hs = (4, 8, 16, 64, 128)[rng.next_below(5)]
        q = [_next_signed(rng) for _ in range(hs)]
        k = [_next_signed(rng) for _ in range(hs)]
        a, b = rng.next_below(4097), rng.next_below(4097)
        shift = rng.next_below(4097 - max(a, b))
        d = abs(_rope_relative_score(q, k, a, b, cfg.rope_base)
                - _rope_relative_score(q, k, a + shift, b + shift, cfg.rope_base))
        worst = max(worst, d)
        if d > 1e-9:
            lines.append(f"FAIL rope shift invariance: diff {d:g} at a={a} b={b} shift={shift} head_size={hs}")
            repro(opts.seed)
            return 1, lines
    lines.append(f"ok rope shift invariance ({opts.rope_cases} cases, worst {worst:g})")

    # -- KV round trip + error paths (turbokv_main.cpp:455-507): store pages == assembled (unrotated) K/V bitwise;
    # a TKVC file with another fingerprint is StaleCacheError, a truncated one FormatError, a missing id NotFound
    rng = SplitMix64(opts.seed ^ 0x57083)
    tmp = tmp_dir or tempfile.mkdtemp(prefix="turbokv-verify-")
    for _ in range(10):
        cid = engine.ingest_chunk_payload("roundtrip", encode(_random_text(rng, 1 + rng.next_below(64))))
        with engine.assemble([cid], T.PositionMode.Reordered) as direct:
            for layer in range(cfg.layer_num):
                for which in ("k", "v"):
                    if not np.array_equal(engine.store_read(cid, layer, which),
                                          direct.read_kv(layer, which, rotated=False)):
                        lines.append(f"FAIL kv round trip: layer {layer} not bit-identical")
                        repro(opts.seed)
                        return 1, lines
        path = os.path.join(tmp, f"{cid:016x}.tkvc")
        engine.export_tkvc(cid, path)
        raw = bytearray(open(path, "rb").read())
        raw[28:36] = struct.pack("<Q", struct.unpack_from("<Q", raw, 28)[0] ^ 1)
        open(path, "wb").write(bytes(raw))
        engine.store_evict(cid)
        try:
            engine.import_tkvc(path)
            lines.append("FAIL kv round trip: stale fingerprint accepted")
            repro(opts.seed)
            return 1, lines
        except T.StaleCacheError:
            pass
    cid = engine.ingest_chunk_payload("roundtrip", encode(_random_text(rng, 32)))
    path = os.path.join(tmp, f"{cid:016x}.tkvc")
    engine.export_tkvc(cid, path)
    raw = open(path, "rb").read()
    open(path, "wb").write(raw[: len(raw) // 2])
    engine.store_evict(cid)
    try:
        engine.import_tkvc(path)
        lines.append("FAIL kv round trip: truncated file accepted")
        repro(opts.seed)
        return 1, lines
    except T.FormatError:
        pass
    try:
        engine.assemble([0xDEADDEADDEADDEAD]).close()
        lines.append("FAIL kv round trip: missing chunk loaded")
        repro(opts.seed)
        return 1, lines
    except T.NotFoundError:
        pass
    lines.append("ok kv round trip (10 cases + error paths)")

    # -- incremental forward (turbokv_main.cpp:509-553): a causal prefill split in two equals the one-shot prefill
    # (last-row logits: the engine returns TTFT logits, not every row's)
    rng = SplitMix64(opts.seed ^ 0x19C8)
    for _ in range(10):
        total = 2 + rng.next_below(95)
        split = 1 + rng.next_below(total - 1)
        tokens = np.array([rng.next_below(cfg.vocab_size) for _ in range(total)], np.int32)
        with engine.assemble([]) as one:
            a = engine.prefill_query(one, tokens)[0]
        with engine.assemble([]) as two:
            engine.prefill_query(two, tokens[:split])
            b = engine.prefill_query(two, tokens[split:])[0]
        diff = _max_abs_diff(a, b)
        if diff > rel * max(float(np.abs(a).max()), 1e-30):
            lines.append(f"FAIL incremental forward: diff {diff:g} (total {total}, split {split})")
            repro(opts.seed)
            return 1, lines
    lines.append("ok incremental forward (10 splits)")

    # -- single-chunk degeneracy (turbokv_main.cpp:555-584): all four paths agree
    rng = SplitMix64(opts.seed ^ 0x51C6)
    for _ in range(5):
        cid = engine.ingest_chunk_payload("single", encode(_random_text(rng, 1 + rng.next_below(64))))
        query = encode(_random_text(rng, 1 + rng.next_below(16)))
        outs = []
        for mode in (T.PositionMode.Reordered, T.PositionMode.Composite):
            with engine.assemble([cid], mode) as c:
                outs.append(engine.prefill_query(c, query)[0])
        for mode in (T.MaskMode.Causal, T.MaskMode.Independent):
            with naive_ids([cid], query, mode) as c:
                outs.append(c.last_logits)
        spread = max(_max_abs_diff(outs[0], o) for o in outs[1:])
        if spread > rel * max(float(np.abs(outs[0]).max()), 1e-30):
            lines.append(f"FAIL single-chunk degeneracy: spread {spread:g}")
            repro(opts.seed)
            return 1, lines
    lines.append("ok single-chunk degeneracy (5 cases)")
    lines.append("all properties hold")
    return 0, lines


def _splitmix_at(seed: int, i: int) -> int:
    """SplitMix64::at(seed, i) (rng.hpp): the i-th draw of the stream seeded with `seed`."""
    from .bench_api import SplitMix64

    r = SplitMix64((seed + i * 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
    return r.next()


def _next_signed(rng) -> float:
    """SplitMix64::next_signed (rng.hpp): 2 * (next() >> 11) * 2^-53 - 1."""
    return 2.0 * ((rng.next() >> 11) * (1.0 / (1 << 53))) - 1.0
