"""Back-to-back rate of the small batch-1 projection GEMMs (QKV, O) over split-K counts (tkv_debug_gemm_bench)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T

L = T.lib()
for name, (M, N, K) in {"qkv": (64, 4608, 3584), "o": (64, 3584, 3584)}.items():
    for sp in (4, 6, 8, 10, 12, 14, 16):
        ms = C.c_double()
        T._check(L.tkv_debug_gemm_bench(0, M, N, K, sp, 0, 100, C.byref(ms)))
        print(f"{name:4s} splits={sp:2d}: {ms.value * 1e3:6.2f} us, {N * K * 2 / (ms.value / 1e3) / 1e9:5.0f} GB/s")
