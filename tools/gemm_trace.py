"""Per-stage pipeline trace of CTA 0 of one tcgen05 GEMM (tkv_debug_gemm_trace): producer issue / MMA-saw-full /
MMA-commit clock64 stamps, summarised as cycles between consecutive stages and producer-vs-MMA slack.
usage: python tools/gemm_trace.py M N K splits swiglu stages smem_kb ctas_per_sm"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T

L = T.lib()
M, N, K, sp, sw, st, smk, cps = (int(v) for v in sys.argv[1:9])
T._check(L.tkv_debug_set_gemm_knobs(st, smk, cps, 1))
ms = C.c_double()
T._check(L.tkv_debug_gemm_bench(0, M, N, K, sp, sw, 5, C.byref(ms)))  # warm
T._check(L.tkv_debug_gemm_trace(1, None, 0))
T._check(L.tkv_debug_gemm_bench(0, M, N, K, sp, sw, 2, C.byref(ms)))  # + 3 warm-up launches inside: last two traced
buf = np.zeros(3 * 1024 + 128 + 256 + 32 + 4096, np.uint64)
T._check(L.tkv_debug_gemm_trace(0, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size))
st3 = buf[:3072].reshape(1024, 3).astype(np.int64)
n = int((st3[:, 1] > 0).sum())
st3 = st3[:n]
t0 = st3[st3 > 0].min()
rel = (st3 - t0)
full = rel[:, 1]
print(f"M={M} N={N} K={K} splits={sp} swiglu={sw} stages={st} smem={smk} cps={cps}: {ms.value*1e3:.2f} us/launch, CTA0 {n} stages")
d = np.diff(full)
print(f"  MMA-saw-full interval: median {np.median(d):.0f} cyc, mean {d.mean():.0f}, p90 {np.percentile(d, 90):.0f}")
if (st3[:, 2] > 0).all():
    print(f"  MMA issue cost (commit - full): median {np.median(rel[:, 2] - rel[:, 1]):.0f} cyc")
iss = rel[:, 0]
valid = iss > 0
lat = (full - iss)[valid]
if len(lat):
    print(f"  producer issue -> full (load latency incl. queueing): median {np.median(lat):.0f} cyc, min {lat.min()}, max {lat.max()}")
print("  MMA saw stages full at:", [int(x) for x in full[:16]])
u = buf[3072:3072 + 128].reshape(64, 2).astype(np.int64)
mm = buf[3200:3456].reshape(64, 4).astype(np.int64)
for r in range(min(8, n), min(12, n)):
    print(f'  stage {r}: full {int(rel[r, 1])} mma-issued', [int(x - t0) for x in mm[r]], 'commit', int(rel[r, 2]))
u = u[u[:, 0] > 0] - t0
print("  epilogue per unit (start, end):", [tuple(int(x) for x in r) for r in u[:8]])
ep = buf[3072 + 384:].astype(np.int64)
print("  epilogue stamps:", [int(x - t0) if x else 0 for x in ep[:24]])
print(f"  last stage full at {int(full[-1])} cyc")

cta = buf[3072 + 384 + 32:].reshape(2, 1024, 2).astype(np.int64)
for par in range(2):
    c = cta[par]
    c = c[c[:, 0] > 0]
    if len(c):
        base = cta[:, :, 0][cta[:, :, 0] > 0].min()
        st, en = (c[:, 0] - base) / 1e3, (c[:, 1] - base) / 1e3
        print(f"  launch parity {par}: {len(c)} CTAs, entry min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f} us, "
              f"exit min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us")
