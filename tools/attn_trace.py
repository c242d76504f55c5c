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
out = np.zeros(512 + 2048, np.uint64)
T._check(L.tkv_debug_attn_trace(0, out.ctypes.data_as(T.U64P), 512 + 2048))
ev = out[:512].reshape(32, 16).astype(np.int64)
cta = out[512:].reshape(1024, 2).astype(np.int64)
cta = cta[cta[:, 0] > 0]
if len(cta):
    s0 = cta[:, 0].min()
    st, en = (cta[:, 0] - s0) / 1e3, (cta[:, 1] - s0) / 1e3
    print(f"{len(cta)} CTAs: start spread {st.max():.2f} us, end min/median/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us, "
          f"duration min/median/max {(en-st).min():.2f}/{np.median(en-st):.2f}/{(en-st).max():.2f} us")
    order = np.argsort(st)
    print("start times (us) by launch index, every 12th:", np.round(st[::12], 2).tolist())
t0 = ev[ev > 0].min()
names = ["h0:S ready", "h0:P released", "hN:S ready", "hN:P released", "mma:PV(j) issued", "mma:S(j) issued",
         "tma:K(j) issue", "tma:V(j) issue", "mma:Q ready", "-", "t0:ld done", "t0:max xchg", "t0:exp c0", "t0:arrive c0",
         "t0:exp c1", "t0:arrive c1"]
EV = [0, 10, 11, 12, 13, 14, 15, 1, 2, 3, 5, 4, 6, 7, 8]
print("kernel entry at", ev[0, 9] - t0, "cycles")
print("previous kernel done (softmax pdl_wait returned) %d, Q staged %d" % (ev[30, 3] - t0, ev[30, 5] - t0))
print("epilogue: o_done seen %d, staged %d, copied out %d, (m, l) written %d" % (ev[31, 0] - t0, ev[31, 5] - t0, ev[31, 6] - t0, ev[31, 1] - t0))
print("cycles since first event (CTA 0); rows = KV tile j")
print("j  " + " ".join(f"{names[e][-13:]:>13s}" for e in EV))
for j in range(30):
    if (ev[j, :16] == 0).all():
        continue
    print(f"{j:<2d} " + " ".join(f"{(ev[j, e] - t0) if ev[j, e] else -1:13d}" for e in EV))
