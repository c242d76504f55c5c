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

