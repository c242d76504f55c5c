"""clock64 timeline of one attention launch INSIDE the C2 turbo forward (layer TKV_TRACE_LAYER, default 14):
the engine context (PDL overlap with the QKV epilogue, K/V from HBM) rather than the standalone kernel."""
import os
import sys

import numpy as np

os.environ.setdefault("TKV_TRACE_LAYER", "14")
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_07590_b200 import turbokv as T  # noqa: E402

cfg = T.ModelConfig.qwen2_7b_like()
eng = T.Engine(cfg, bench.SEED, dtype="bf16", store_capacity_tokens=bench.N_CHUNKS * bench.CHUNK_TOKENS * 2)
payloads, query = bench.workload()
ids = eng.ingest_chunks(payloads)
L = T.lib()
for _ in range(3):
    with eng.assemble(ids, T.PositionMode.Reordered) as ctx:
        eng.prefill_query(ctx, query)
out = np.zeros(512 + 2048, np.uint64)
T._check(L.tkv_debug_attn_trace(0, out.ctypes.data_as(T.U64P), 512 + 2048))
ev = out[:512].reshape(32, 16).astype(np.int64)
cta = out[512:].reshape(1024, 2).astype(np.int64)
# this launch's CTAs (the single-request split-K grid: Hkv x s_c CTAs of the compact last tile, then the
# (gx - 1) x Hkv x s full-tile CTAs; the rest of the buffer may hold other launches' stamps)
NCTA, NCOMP = int(os.environ.get("C2_CTAS", 148)), int(os.environ.get("C2_COMPACT_CTAS", 28))
cta = cta[:NCTA]
s0 = cta[:, 0].min()
st, en = (cta[:, 0] - s0) / 1e3, (cta[:, 1] - s0) / 1e3
dur = en - st
print(f"layer {os.environ['TKV_TRACE_LAYER']}: {len(cta)} CTAs, start spread {st.max():.2f} us, "
      f"end min/median/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us")
print("CTA duration us, compact tile min/median/max %.2f/%.2f/%.2f, full tiles %.2f/%.2f/%.2f"
      % (dur[:NCOMP].min(), np.median(dur[:NCOMP]), dur[:NCOMP].max(), dur[NCOMP:].min(), np.median(dur[NCOMP:]),
         dur[NCOMP:].max()))
t0 = ev[0, 9]
names = ["smA:S ready", "smA:P arrive", "smB:S ready", "smB:P arrive", "mma:PV_A issued", "mma:PV_B issued",
         "tma:K(j) issue", "tma:V(j) issue", "mma:Q ready"]
if ev[31, 7] > 0 and ev[31, 1] > 0:
    print("CTA 0 entry -> partials written: %d cycles in %.2f us = %.2f GHz; CTA 0 exit %.2f us after entry"
          % (ev[31, 1] - ev[0, 9], (ev[31, 7] - cta[0, 0]) / 1e3, (ev[31, 1] - ev[0, 9]) / (ev[31, 7] - cta[0, 0]),
             (cta[0, 1] - cta[0, 0]) / 1e3))
print("cycles since CTA (0,0,0) entry")
print("previous kernel done (softmax pdl_wait returned) %d, Q loads back %d, Q staged %d"
      % (ev[30, 3] - t0, ev[30, 4] - t0, ev[30, 5] - t0))
print("epilogue: o_done %d, partials written %d" % (ev[31, 0] - t0, ev[31, 1] - t0))
print("j   " + " ".join(f"{n:>16s}" for n in names))
for j in range(30):
    if (ev[j, :9] == 0).all():
        continue
    print(f"{j:<3d} " + " ".join(f"{(ev[j, e] - t0) if ev[j, e] else -1:16d}" for e in range(9)))
print("CTA start / duration us by launch index:")
for b in range(0, len(cta), 4):
    print("  " + "  ".join(f"{b + i:3d}: {st[b + i]:5.2f}+{dur[b + i]:5.2f}" for i in range(4) if b + i < len(cta)))
