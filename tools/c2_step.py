"""C2 turbo step timing for knob sweeps (TUNING builds read TKV_* knobs): p50 / mean TTFT over N steps."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_07590_b200 import turbokv as T  # noqa: E402


def main(steps=30, flags=0):
    cfg = T.ModelConfig.qwen2_7b_like()
    eng = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=16 * 512 * 2, flags=flags, exact_fingerprint=0)
    payloads, query = bench.workload()
    ids = eng.ingest_chunks(payloads)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=dev)
    dq = torch.from_numpy(query).to(dev)
    dl = torch.empty(cfg.vocab_size, dtype=torch.float32, device=dev)

    def step():
        ctx = eng.assemble(ids, T.PositionMode.Reordered)
        eng.prefill_query_device(ctx, dq.data_ptr(), len(query), dl.data_ptr())
        ctx.close()

    for _ in range(5):
        step()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"flags={flags} env={ {k: v for k, v in os.environ.items() if k.startswith('TKV_')} } "
          f"p50 {statistics.median(ts):.3f} ms mean {statistics.mean(ts):.3f} ms logit0 {dl[0].item():.6f}")


if __name__ == "__main__":
    main(flags=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
