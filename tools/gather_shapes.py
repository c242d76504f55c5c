"""KV gather (assemble) time per launch, in the chain (tkv_kernel_timeline), for different chunk shapes / context
sizes at Qwen2-7B dims: where does the C3 gather (20 x 800-token chunks) lose bandwidth against C2 (16 x 512)?"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T  # noqa: E402

cfg = T.ModelConfig.qwen2_7b_like()
eng = T.Engine(cfg, 42, dtype="bf16", store_capacity_tokens=200 * 1024, exact_fingerprint=0)
rng = np.random.default_rng(5)
corpus = {}
for L in (512, 800, 1024):
    corpus[L] = eng.ingest_chunks([rng.integers(97, 123, L - 2).astype(np.int32) for _ in range(40)])
kvb = cfg.layer_num * 2 * cfg.kv_dim * 2
for L, n, reuse in [(512, 16, True), (800, 20, True), (800, 20, False), (512, 32, True), (1024, 16, True), (800, 10, True)]:
    ids = corpus[L][:n]
    held = []
    for _ in range(3):
        c = eng.assemble(ids)
        (c.close() if reuse else held.append(c))
    eng.kernel_timeline(True)
    for _ in range(5):
        c = eng.assemble(ids)
        (c.close() if reuse else held.append(c))
    torch.cuda.synchronize()
    tl, cls = eng.kernel_timeline(False)
    d = (tl[:, 1] - tl[:, 0])[cls == 0] / 1e3
    byts = 2 * n * L * kvb
    print(f"{n:3d} x {L:4d} tokens, caches {'recycled' if reuse else 'fresh    '}: gather {np.median(d):7.1f} us "
          f"= {byts / np.median(d) / 1e6:5.2f} TB/s")
    for c in held:
        c.close()
