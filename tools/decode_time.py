"""Time the decode-sized attention kernels on the C2 last-layer shape (1 row, 8256 keys) and a greedy decode."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T

H, Hkv, d, Tk = 28, 4, 128, 8256
rng = np.random.default_rng(0)
q = rng.uniform(-1, 1, (1, H * d)).astype(np.float32)
k = rng.uniform(-1, 1, (Tk, Hkv * d)).astype(np.float32)
lo, hi = np.zeros(1, np.int32), np.array([Tk - 1], np.int32)
import os
os.environ.setdefault("TKV_DEBUG_TIME_ITERS", "0")
for impl in (0, 2):
    T.debug_attention(q, k, k, lo, hi, H, Hkv, d, dtype="bf16", impl=impl)
print("ok")
