#!/bin/bash
# A/B engine flags (tkv.h TKV_FLAG_*) through the C2 turbo step: p50 TTFT.
for f in "$@"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --turbo-only --flags $f 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flags', $f, round(d['p50_ttft_ms'],3))"
done
