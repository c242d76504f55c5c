#!/bin/bash
# A/B an environment knob through the C2 turbo step: tools/env_bench.sh VAR v1 v2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --turbo-only 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var', '$v', round(d['p50_ttft_ms'],3))"
done
