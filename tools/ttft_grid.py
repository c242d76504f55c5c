"""`turbokv bench` (tools/turbokv_main.cpp:666-710) on the B200 engine: the reference's TTFT grid through
bench_api.run_bench -- CSV (docs/formats.md "bench CSV") on stdout, medians per (doc_tokens, path) on stderr.
  python tools/ttft_grid.py [--preset toy|qwen2-7b] [--doc-grid 512,1024,2048,4096] [--reps 5] [--query-tokens 64]
"""
import argparse
import sys

sys.path.insert(0, ".")
from paper_2410_07590_b200 import bench_api as B  # noqa: E402
from paper_2410_07590_b200 import turbokv as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="toy", choices=["toy", "qwen2-7b"])
ap.add_argument("--doc-grid", default="512,1024,2048,4096")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--query-tokens", type=int, default=64)
ap.add_argument("--seed", type=int, default=42)
ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
a = ap.parse_args()
cfg = T.ModelConfig.toy() if a.preset == "toy" else T.ModelConfig.qwen2_7b_like()
config = B.BenchConfig(doc_grid=sorted(int(x) for x in a.doc_grid.split(",")), query_tokens=a.query_tokens,
                       reps=a.reps, seed=a.seed)
eng = T.Engine(cfg, a.seed, dtype=a.dtype, store_capacity_tokens=max(config.doc_grid) * 2 + 4096)
rows = B.run_bench(eng, config)
sys.stdout.write(B.bench_csv(rows))
for s in B.summarize(rows):
    print(f"doc_tokens={s.doc_tokens} turbo_median_ms={s.turbo_median_ms:.3f} naive_median_ms={s.naive_median_ms:.3f} "
          f"speedup={s.speedup:.1f}x", file=sys.stderr)
