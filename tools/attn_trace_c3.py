"""CTA timeline of the batched attention launch of one layer (TKV_TRACE_LAYER, default 14) in a C3-shaped
batched prefill: 32 requests x (20 chunks x 800 tokens) + 64-token queries, Qwen2-7B shape."""
import os
import sys

import numpy as np

os.environ.setdefault("TKV_TRACE_LAYER", "14")
sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T  # noqa: E402

B, NC, CT, CORPUS, Q = int(os.environ.get("C3_BATCH", 32)), 20, 800, 160, 64
cfg = T.ModelConfig.qwen2_7b_like()
eng = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=CORPUS * 1024 + 65536)
rng = np.random.default_rng(0xC3)
cids = eng.ingest_chunks([rng.integers(97, 123, CT - 2).astype(np.int32) for _ in range(CORPUS)])
picks = [rng.choice(CORPUS, NC, replace=False) for _ in range(B)]
queries = [rng.integers(97, 123, Q).astype(np.int32) for _ in range(B)]
L = T.lib()
for _ in range(2):
    ctxs = [eng.assemble([cids[j] for j in pk], T.PositionMode.Reordered) for pk in picks]
    eng.prefill_query_batch(ctxs, queries)
    for c in ctxs:
        c.close()
out = np.zeros(512 + 2048, np.uint64)
T._check(L.tkv_debug_attn_trace(0, out.ctypes.data_as(T.U64P), 512 + 2048))
ev = out[:512].reshape(32, 16).astype(np.int64)
cta = out[512:].reshape(1024, 2).astype(np.int64)
ncta = ((Q * 7 + 127) // 128) * 4 * B  # this launch's grid (row tiles x kv heads x requests), no split-K
cta = cta[:ncta]
cta = cta[cta[:, 0] > 0]
s0 = cta[:, 0].min()
st, en = (cta[:, 0] - s0) / 1e3, (cta[:, 1] - s0) / 1e3
dur = en - st
print(f"{len(cta)} CTAs: kernel span {en.max():.1f} us; start times: first-wave {np.sort(st)[:148].max():.1f} us, "
      f"last {st.max():.1f} us; duration min/median/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us")
print("sum of CTA durations / (148 x span) = %.3f" % (dur.sum() / (148 * en.max())))
for q in (0.1, 0.5, 0.9, 1.0):
    print(f"  end time quantile {q}: {np.quantile(en, q):.1f} us")
print("duration by linear CTA index (every 16th):", np.round(dur[::16], 1).tolist())
t0 = ev[0, 9]
print("CTA 0: entry->Q staged %d, first S ready %d, o_done %d cycles" % (ev[30, 5] - t0, ev[0, 0] - t0, ev[31, 0] - t0))
s_ready = ev[:30, 0]
per = np.diff(s_ready[s_ready > 0])
print("per-tile period (S ready to S ready), cycles: median %d, tiles 1-29: %s" % (np.median(per), per.tolist()))
sm = ev[:30, 1] - ev[:30, 0]
print("softmax S ready -> P released, cycles: median %d" % np.median(sm[ev[:30, 1] > 0]))
# per-tile event table of CTA 0 (cycles relative to this tile's S-ready): K / V TMA issued, MMA warp past the K wait,
# S MMAs issued, MMA warp past the last P chunk wait, PV MMAs
# issued, S loaded from TMEM, row max done, first P chunk stored / released, all P released
names = {6: "K issued", 7: "V issued", 14: "K ready@mma", 5: "S issued", 15: "P3 seen@mma", 4: "PV issued", 10: "S loaded", 11: "max", 12: "P0 stored",
         13: "P0 released", 1: "P released"}
print("tile " + " ".join(f"{v:>11s}" for v in names.values()))
for j in range(8, 16):
    print(f"{j:4d} " + " ".join(f"{ev[j, e] - ev[j, 0]:11d}" if ev[j, e] > 0 else f"{'-':>11s}" for e in names))
