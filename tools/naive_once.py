"""One full-concat prefill of the C2 request (16 x 512 chunks + 64-token query, Qwen2-7B shape, bf16): the
large-M (8256-token) GEMM / attention path, for ncu captures."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_07590_b200 import turbokv as T  # noqa: E402

import numpy as np  # noqa: E402

cfg = T.ModelConfig.qwen2_7b_like()
eng = T.Engine(cfg, bench.SEED, dtype="bf16", store_capacity_tokens=bench.N_CHUNKS * bench.CHUNK_TOKENS * 2)
payloads, query = bench.workload()
framed = [np.concatenate([[256], p, [257]]).astype(np.int32) for p in payloads]
eng.naive_prefill(framed, query, T.MaskMode.Causal, keep_context=False)
print("ok")
