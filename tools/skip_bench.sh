#!/bin/bash
# Cost attribution: TTFT with kernel classes dropped (TKV_TIMING_SKIP bitmask; results numerically invalid).
# 1 = residual after O-proj, 2 = residual after down-proj, 4 = qkv epilogue, 8 = attention
for m in "$@"; do
  TKV_TIMING_SKIP=$m timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --naive-reps 1 --turbo-only 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip', $m, round(d['p50_ttft_ms'],3))"
done
