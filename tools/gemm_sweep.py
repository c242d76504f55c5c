"""Sweep tcgen05 GEMM knobs on the C2 per-layer projection shapes (64 tokens). Prints achieved weight GB/s."""
import ctypes as C
import itertools
import json
import sys

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T

L = T.lib()
SHAPES = {"qkv": (64, 4608, 3584, 4, 0), "o": (64, 3584, 3584, 5, 0), "gu": (64, 37888, 3584, 1, 1),
          "down": (64, 3584, 18944, 5, 0)}
res = []
for stages, smem, cps, ef in itertools.product([4, 6, 8], [200, 224], [1, 2], [1, 0]):
    if cps == 2 and smem > 112:
        smem_eff = 110
    else:
        smem_eff = smem
    T._check(L.tkv_debug_set_gemm_knobs(stages, smem_eff, cps, ef))
    row = {"stages": stages, "smem_kb": smem_eff, "ctas_per_sm": cps, "evict_first": ef}
    for name, (M, N, K, sp, sw) in SHAPES.items():
        ms = C.c_double()
        rc = L.tkv_debug_gemm_bench(0, M, N, K, sp, sw, 50, C.byref(ms))
        row[name] = round(N * K * 2 / (ms.value / 1e3) / 1e9, 1) if rc == 0 else None
    row["layer_us"] = round(sum(SHAPES[n][1] * SHAPES[n][2] * 2 / (row[n] * 1e9) * 1e6 for n in SHAPES if row[n]), 1)
    print(json.dumps(row), flush=True)
    res.append(row)
best = min(res, key=lambda r: r["layer_us"])
print("BEST", json.dumps(best))
