#!/bin/bash
# A/B the attention-time L2 weight prefetch amount (TKV_L2_PREFETCH_MB) through the C2 bench.
for mb in "$@"; do
  TKV_L2_PREFETCH_MB=$mb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --naive-reps 1 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf', $mb, round(d['p50_ttft_ms'],3), {k: round(v,3) for k,v in d['device_ms_per_step'].items()})"
done
