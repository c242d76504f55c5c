#!/bin/bash
# A/B GEMM knobs (TKV_GEMM_KNOBS="stages,smem_kb,ctas_per_sm,evict_first") through the C2 turbo step.
for k in "$@"; do
  TKV_GEMM_KNOBS=$k timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --naive-reps 1 --turbo-only 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('knobs', '$k', round(d['p50_ttft_ms'],3))"
done
