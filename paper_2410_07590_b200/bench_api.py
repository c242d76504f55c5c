"""The reference's TTFT benchmark API (include/turbokv/bench.hpp, src/bench.cpp) over the B200 engine.

Same names, arguments, corpus, query, windows and CSV/summary formats, so the reference's bench callers
(`turbokv bench`, acceptance_main.cpp check_ttft) read this engine's numbers unchanged:
  * ingest_synthetic (bench.cpp:36-66): chunk_count = max(doc_grid) / 64 chunks; chunk i's payload is
    random_word(rng, 61) + " " with ONE SplitMix64 stream seeded by config.seed (62 payload bytes = 64 framed
    tokens), ingested in one batched block-diagonal forward (chunk ids are content addresses).
  * run_bench (bench.cpp:68-111): query = random_word(SplitMix64(seed ^ 0x51DEC0DE), query_tokens); per grid
    point the first doc_tokens / 64 chunks; turbo window = assemble + prefill_query (cache load inside the
    window), naive window = naive_prefill(framed chunks, Independent) with the tokens already in hand; one
    warm-up repetition (rep -1) per (grid point, path) discarded; FlopCounter totals per row.
  * bench_csv / summarize (bench.cpp:113-138): header `doc_tokens,query_tokens,path,rep,ttft_ms,measured_flops`,
    doubles in C++ default stream formatting (6 significant digits); medians per (doc_tokens, path).
Wall-clock windows (time.perf_counter) like the reference's steady_clock; every engine call returns with its
host-side results (logits in host memory), so a window ends when the first-token logits are on the host.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import turbokv as T

K_BENCH_CHUNK_TOKENS = 64  # bench.hpp:29
_M64 = (1 << 64) - 1
_PHI = 0x9E3779B97F4A7C15


class SplitMix64:
    """include/turbokv/rng.hpp:10-40 (stateful stream; next() == SplitMix64::at(seed, i) for the i-th draw)."""

    def __init__(self, seed: int):
        self.state = seed & _M64

    def next(self) -> int:
        self.state = (self.state + _PHI) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def next_below(self, n: int) -> int:
        return self.next() % n


def random_word(rng: SplitMix64, n: int) -> str:
    """bench.cpp:21-25"""
    return "".join(chr(ord("a") + rng.next_below(26)) for _ in range(n))


def encode(text: str) -> np.ndarray:
    """tok::encode (tokenizer.cpp): one token per byte."""
    return np.frombuffer(text.encode("utf-8"), np.uint8).astype(np.int32)


@dataclass
class BenchConfig:
    """bench.hpp:11-16"""
    doc_grid: list = field(default_factory=list)  # framed chunk-token totals, ascending
    query_tokens: int = 64
    reps: int = 5
    seed: int = 42


@dataclass
class BenchRow:
    """bench.hpp:18-25"""
    doc_tokens: int
    query_tokens: int
    path: str
    rep: int
    ttft_ms: float
    measured_flops: int


@dataclass
class BenchSummary:
    """bench.hpp:45-50"""
    doc_tokens: int
    turbo_median_ms: float
    naive_median_ms: float
    speedup: float


def synthetic_payloads(config: BenchConfig) -> list:
    """The payloads ingest_synthetic feeds the engine (validation as bench.cpp:37-47)."""
    if not config.doc_grid:
        raise T.DomainError("bench: empty doc grid")
    for d in config.doc_grid:
        if d < K_BENCH_CHUNK_TOKENS or d % K_BENCH_CHUNK_TOKENS:
            raise T.DomainError(f"bench: grid entries must be positive multiples of {K_BENCH_CHUNK_TOKENS}")
    rng = SplitMix64(config.seed)
    count = max(config.doc_grid) // K_BENCH_CHUNK_TOKENS
    # 61 letters + trailing space = 62 payload bytes = 64 framed tokens
    return [encode(random_word(rng, K_BENCH_CHUNK_TOKENS - 3) + " ") for _ in range(count)]


def ingest_synthetic(engine: T.Engine, config: BenchConfig) -> list:
    """bench.cpp:36-66: returns the chunk ids in ingest order."""
    payloads = synthetic_payloads(config)
    return engine.ingest_chunks(payloads)


def bench_query(config: BenchConfig) -> np.ndarray:
    """bench.cpp:74-76"""
    return encode(random_word(SplitMix64(config.seed ^ 0x51DEC0DE), config.query_tokens))


def run_bench(engine: T.Engine, config: BenchConfig) -> list:
    """bench.cpp:68-111"""
    if config.reps < 1:
        raise T.DomainError("bench: reps must be >= 1")
    if config.query_tokens < 1:
        raise T.DomainError("bench: query_tokens must be >= 1")
    payloads = synthetic_payloads(config)
    ids = engine.ingest_chunks(payloads)
    framed_all = [np.concatenate([[256], p, [257]]).astype(np.int32) for p in payloads]
    query = bench_query(config)
    rows = []
    for doc_tokens in config.doc_grid:
        n = doc_tokens // K_BENCH_CHUNK_TOKENS
        subset, framed = ids[:n], framed_all[:n]
        for rep in range(-1, config.reps):  # rep -1 is the warm-up and is not recorded
            counter = T.FlopCounter()
            t0 = time.perf_counter()
            with engine.assemble(subset, T.PositionMode.Reordered) as ctx:
                engine.prefill_query(ctx, query, counter)
                elapsed = (time.perf_counter() - t0) * 1e3
            if rep >= 0:
                rows.append(BenchRow(doc_tokens, config.query_tokens, "turbo-reordered", rep, elapsed,
                                     counter.total()))
        for rep in range(-1, config.reps):
            counter = T.FlopCounter()
            t0 = time.perf_counter()
            engine.naive_prefill(framed, query, T.MaskMode.Independent, counter, keep_context=False)
            elapsed = (time.perf_counter() - t0) * 1e3
            if rep >= 0:
                rows.append(BenchRow(doc_tokens, config.query_tokens, "naive-independent", rep, elapsed,
                                     counter.total()))
    return rows


def _cxx_double(x: float) -> str:
    """operator<< on a double with the default stream state (6 significant digits, %g style)."""
    return "%g" % x


def bench_csv(rows) -> str:
    """bench.cpp:113-121"""
    out = ["doc_tokens,query_tokens,path,rep,ttft_ms,measured_flops"]
    out += [f"{r.doc_tokens},{r.query_tokens},{r.path},{r.rep},{_cxx_double(r.ttft_ms)},{r.measured_flops}"
            for r in rows]
    return "\n".join(out) + "\n"


def _median(xs) -> float:
    """bench.cpp:27-32"""
    xs = sorted(xs)
    n = len(xs)
    if n == 0:
        raise T.DomainError("median of empty sample")
    return xs[n // 2] if n % 2 == 1 else 0.5 * (xs[n // 2 - 1] + xs[n // 2])


def summarize(rows) -> list:
    """bench.cpp:123-138: medians per (doc_tokens, path), ascending doc_tokens."""
    grouped: dict = {}
    for r in rows:
        grouped.setdefault(r.doc_tokens, {}).setdefault(r.path, []).append(r.ttft_ms)
    out = []
    for d in sorted(grouped):
        by = grouped[d]
        if "turbo-reordered" not in by or "naive-independent" not in by:
            raise T.DomainError(f"bench: doc_tokens {d} lacks one of the two paths")  # map::at throws
        t, nv = _median(by["turbo-reordered"]), _median(by["naive-independent"])
        out.append(BenchSummary(d, t, nv, nv / t))
    return out
