"""Timeline of one attention CTA (C2 query prefill shape) from clock64 stamps (tkv_debug_attn_trace)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T

L = T.lib()
P, Q, H, Hkv, d = 8192, 64, 28, 4, 128
rng = np.random.default_rng(0)
q = rng.uniform(-1, 1, (Q, H * d)).astype(np.float32)
k = rng.uniform(-1, 1, (P + Q, Hkv * d)).astype(np.float32)
v = rng.uniform(-1, 1, (P + Q, Hkv * d)).astype(np.float32)
lo = np.zeros(Q, np.int32)
hi = (P + np.arange(Q)).astype(np.int32)
T._check(L.tkv_debug_attn_trace(1, None, 0))
for _ in range(3):
    T.debug_attention(q, k, v, lo, hi, H, Hkv, d, dtype="bf16")
out = np.zeros(320, np.uint64)
T._check(L.tkv_debug_attn_trace(0, out.ctypes.data_as(T.U64P), 320))
ev = out.reshape(32, 10).astype(np.int64)
t0 = ev[ev > 0].min()
names = ["sm:S ready", "sm:pass1+bar", "sm:O(j-1) ready", "sm:P arrive", "mma:P seen", "mma:PV issued",
         "mma:S(j) issued", "tma:K(j) issue", "tma:V(j) issue"]
print("cycles since first event (CTA 0); rows = KV tile j")
print("j   " + " ".join(f"{n:>16s}" for n in names))
for j in range(32):
    if (ev[j, :9] == 0).all():
        continue
    print(f"{j:<3d} " + " ".join(f"{(ev[j, e] - t0) if ev[j, e] else -1:16d}" for e in range(9)))
