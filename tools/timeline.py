"""In-chain kernel timeline of the C2 turbo step (tkv_kernel_timeline): per-class time per request and the four
projection GEMMs' mean in-chain durations, plus the p50 step. TUNING builds read TKV_* knobs (sweeps)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_07590_b200 import turbokv as T  # noqa: E402


def main(steps=10):
    cfg = T.ModelConfig.qwen2_7b_like()
    c3 = os.environ.get("TL_C3") == "1"  # C3: batch 32 x (20 x 800-token chunks + 64-token query), one step = a batch
    eng = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=(160 * 832 if os.environ.get("TL_C3") == "1" else 64 * 512) + 65536,
                   exact_fingerprint=0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=dev)
    c5 = os.environ.get("TL_C5") == "1"  # C5: one block-diagonal ingest forward of 32 x 512-token chunks = a step
    if c5:
        steps = 3
        rng = np.random.default_rng(0xC5)
        rounds = iter(range(1 << 30))

        def step():
            r = next(rounds)
            pays = [rng.integers(97, 123, 510).astype(np.int32) for _ in range(32)]
            ids = eng.ingest_chunks(pays)
            for i in ids:
                eng.store_evict(i)
    elif c3:
        steps = 2
        rng = np.random.default_rng(0xC3)
        cids = eng.ingest_chunks([rng.integers(97, 123, 798).astype(np.int32) for _ in range(160)])
        picks = [rng.choice(160, 20, replace=False) for _ in range(32)]
        queries = [rng.integers(97, 123, 64).astype(np.int32) for _ in range(32)]

        def step():
            ctxs = [eng.assemble([cids[j] for j in pk], T.PositionMode.Reordered) for pk in picks]
            eng.prefill_query_batch(ctxs, queries)
            for c in ctxs:
                c.close()
    else:
        payloads, query = bench.workload()
        ids = eng.ingest_chunks(payloads)
        dq = torch.from_numpy(query).to(dev)
        dl = torch.empty(cfg.vocab_size, dtype=torch.float32, device=dev)

        def step():
            ctx = eng.assemble(ids, T.PositionMode.Reordered)
            eng.prefill_query_device(ctx, dq.data_ptr(), len(query), dl.data_ptr())
            ctx.close()

    for _ in range(2 if (c3 or c5) else 5):
        step()
    ts = []
    for _ in range(3 if (c3 or c5) else 20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    eng.kernel_timeline(True)
    for _ in range(steps):
        step()
    stream.synchronize()
    tl, cls = eng.kernel_timeline(False)
    dur = np.clip(tl[:, 1] - tl[:, 0], 0, None) / 1e3  # us
    per = {k: dur[cls == i].sum() / steps / 1e3 for i, k in enumerate(T.Engine.TIMELINE_CLASSES)}
    gd = dur[cls == T.Engine.TIMELINE_CLASSES.index("gemm")]
    if len(gd) != steps * cfg.layer_num * 4:
        print(f"{len(gd) / steps:.0f} GEMM launches per step; launches per step {len(tl) / steps:.0f}")
        gd = np.resize(gd, steps * cfg.layer_num * 4)
    g = gd.reshape(steps, cfg.layer_num, 4)[:, :-1]
    # handoff gap between consecutive launches: next first-CTA-past-wait minus previous last-warp-done
    names = T.Engine.TIMELINE_CLASSES
    gaps = {}
    for i in range(1, len(tl)):
        if tl[i, 0] <= 0 or tl[i - 1, 1] <= 0:
            continue
        key = f"{names[cls[i - 1]]}->{names[cls[i]]}"
        gaps.setdefault(key, []).append((tl[i, 0] - tl[i - 1, 1]) / 1e3)
    if os.environ.get("TL_GAPS", "1") == "1":
        for k, v in sorted(gaps.items(), key=lambda kv: -sum(kv[1])):
            print(f"  gap {k:28s} n/step {len(v) / steps:6.1f}  median {np.median(v):6.2f} us  total/step {sum(v) / steps:7.1f} us")
    ep = dur[cls == T.Engine.TIMELINE_CLASSES.index("epilogue")]
    if c5 and len(ep) % steps == 0 and (len(ep) // steps - 2) % 3 == 0:
        # ingest forwards stop after the last layer's K/V: embed, 3 per layer, the last layer's QKV epilogue only
        e5 = ep.reshape(steps, -1)[:, 1:-1].reshape(steps, -1, 3)
        print("  epilogue us per layer: qkv %.1f  residual(O) %.1f  residual(down) %.1f"
              % (e5[..., 0].mean(), e5[..., 1].mean(), e5[..., 2].mean()))
    per_layer = (len(ep) // steps - 1) // cfg.layer_num  # embed, then per layer: QKV epilogue(s), residual x2
    if per_layer >= 3 and len(ep) == steps * (1 + per_layer * cfg.layer_num):
        e = ep.reshape(steps, -1)[:, 1:].reshape(steps, cfg.layer_num, per_layer)
        print("  epilogue us per layer: qkv %.1f  residual(O) %.1f  residual(down) %.1f  (launches/layer %d)"
              % (e[..., :per_layer - 2].sum(-1).mean(), e[..., -2].mean(), e[..., -1].mean(), per_layer))
    at = dur[cls == T.Engine.TIMELINE_CLASSES.index("attention")]
    if len(at) == steps * cfg.layer_num * 2:  # attention, then its split merge, per layer
        a2 = at.reshape(steps, cfg.layer_num, 2)
        print("  attention us per layer: kernel %.2f  merge %.2f" % (a2[..., 0].mean(), a2[..., 1].mean()))
    env = {k: v for k, v in os.environ.items() if k.startswith("TKV_") and k != "TKV_LIB_PATH"}
    print(f"{env} p50 {statistics.median(ts):.3f} ms | in-chain ms: " + " ".join(f"{k} {v:.3f}" for k, v in per.items())
          + f" | gemm us qkv {g[..., 0].mean():.2f} o {g[..., 1].mean():.2f} gate_up {g[..., 2].mean():.2f}"
            f" down {g[..., 3].mean():.2f}")


if __name__ == "__main__":
    main()
