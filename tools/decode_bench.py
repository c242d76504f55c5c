"""Greedy-decode step time on the C2 request (16 x 512-token chunks + 64-token query, Qwen2-7B shape, bf16):
tcgen05 tile attention (default) vs the decode-sized split-K kernel (TKV_FLAG_DECODE_ATTN)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_07590_b200 import turbokv as T  # noqa: E402

NEW = 32
cfg = T.ModelConfig.qwen2_7b_like()
for flags in (0, 0x40, 0, 0x40):  # 0x40 = TKV_FLAG_DECODE_ATTN
    eng = T.Engine(cfg, bench.SEED, dtype="bf16", store_capacity_tokens=bench.N_CHUNKS * bench.CHUNK_TOKENS * 2,
                   flags=flags)
    payloads, query = bench.workload()
    ids = eng.ingest_chunks(payloads)
    ts = []
    for rep in range(4):
        with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
            eng.prefill_query(ctx, query)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            toks = eng.greedy_decode(ctx, NEW)
            torch.cuda.synchronize()
            if rep:
                ts.append((time.perf_counter() - t0) / max(len(toks), 1))
    print(f"flags {flags:#x}: {len(toks)} tokens, {1e3 * sorted(ts)[len(ts) // 2]:.3f} ms per decode step")
    del eng
