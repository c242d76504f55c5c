"""Timeline of one attention CTA (C2 query prefill shape) from clock64 stamps (tkv_debug_attn_trace)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T

L = T.lib()
import os
P, Q, H, Hkv, d = int(os.environ.get("TRACE_P", 8192)), 64, 28, 4, 128
rng = np.random.default_rng(0)
q = rng.uniform(-1, 1, (Q, H * d)).astype(np.float32)
k = rng.uniform(-1, 1, (P + Q, Hkv * d)).astype(np.float32)
v = rng.uniform(-1, 1, (P + Q, Hkv * d)).astype(np.float32)
lo = np.zeros(Q, np.int32)
hi = (P + np.arange(Q)).astype(np.int32)
T._check(L.tkv_debug_attn_trace(1, None, 0))
for _ in range(3):
    T.debug_attention(q, k, v, lo, hi, H, Hkv, d, dtype="bf16")
out = np.zeros(320 + 2048, np.uint64)
T._check(L.tkv_debug_attn_trace(0, out.ctypes.data_as(T.U64P), 320 + 2048))
ev = out[:320].reshape(32, 10).astype(np.int64)
cta = out[320:].reshape(1024, 2).astype(np.int64)
cta = cta[cta[:, 0] > 0]
if len(cta):
    s0 = cta[:, 0].min()
    st, en = (cta[:, 0] - s0) / 1e3, (cta[:, 1] - s0) / 1e3
    print(f"{len(cta)} CTAs: start spread {st.max():.2f} us, end min/median/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us, "
          f"duration min/median/max {(en-st).min():.2f}/{np.median(en-st):.2f}/{(en-st).max():.2f} us")
    order = np.argsort(st)
    print("start times (us) by launch index, every 12th:", np.round(st[::12], 2).tolist())
t0 = ev[ev > 0].min()
import os
names_sm = ["smA:S ready", "smA:P arrive", "smB:S ready", "smB:P arrive", "smA:ld done", "smA:max done", "smA:chunk1", "smA:chunk3", "smA:st done"]
names = ["smA:S ready", "smA:P arrive", "smB:S ready", "smB:P arrive", "mma:PV_A issued", "mma:PV_B issued",
         "tma:K(j) issue", "tma:V(j) issue", "mma:Q ready"]
print("kernel entry at", ev[0, 9] - t0, "cycles")
print("cycles since first event (CTA 0); rows = KV tile j")
if os.environ.get("TRACE_SM") == "1": names = names_sm
if os.environ.get("TRACE_SM") == "2": names = names[:4] + ["mma:P_A seen", "mma:PV_A issued", "mma:K(j+1) seen", "mma:S_A(j+1) iss", "mma:P_B seen"]
print("j   " + " ".join(f"{n:>16s}" for n in names))
print("epilogue: o_done seen %d, partials written %d, grid sync passed %d, merge done %d" % tuple(ev[31, e] - t0 for e in range(4)))
print("  merge: first partial load back %d, old-line load back %d" % (ev[30, 1] - t0, ev[30, 2] - t0))
print("  staged %d, stage barrier %d, copied out %d, merge loads issued %d, merge math done %d" % (ev[31, 4] - t0, ev[31, 5] - t0, ev[31, 6] - t0, ev[30, 0] - t0, ev[31, 7] - t0))
for j in range(30):
    if (ev[j, :9] == 0).all():
        continue
    print(f"{j:<3d} " + " ".join(f"{(ev[j, e] - t0) if ev[j, e] else -1:16d}" for e in range(9)))
