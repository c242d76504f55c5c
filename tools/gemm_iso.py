"""Back-to-back (isolated) tcgen05 GEMM weight-stream rate on the C2 projection shapes at the default knobs
(tkv_debug_gemm_bench: `iters` launches on one stream, PDL-chained, events around all of them)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T

L = T.lib()
SHAPES = {"qkv": (64, 4608, 3584, 8, 0), "o": (64, 3584, 3584, 10, 0), "gate_up": (64, 37888, 3584, 1, 1),
          "down": (64, 3584, 18944, 10, 0)}
for name, (M, N, K, sp, sw) in SHAPES.items():
    ms = C.c_double()
    T._check(L.tkv_debug_gemm_bench(0, M, N, K, sp, sw, 50, C.byref(ms)))
    print(f"{name:8s} N={N:6d} K={K:6d} splits={sp:2d}: {ms.value * 1e3:7.2f} us/launch, "
          f"{N * K * 2 / (ms.value / 1e3) / 1e9:7.0f} GB/s of weights")
