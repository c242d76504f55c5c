#!/bin/bash
# A/B kernel variants (tools/libtkv_*.so built with different compile-time knobs) through the C2 bench.
for so in "$@"; do
  TKV_LIB_PATH=$so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --naive-reps 1 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', round(d['p50_ttft_ms'],3), {k: round(v,3) for k,v in d['device_ms_per_step'].items()})"
done
