#!/bin/bash
# A/B an env knob on the large-M paths: C5 ingest TFLOP/s, C3 batch req/s, full-concat prefill ms (+ C2 TTFT).
var=$1; shift
for v in "$@"; do
  env $var=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --c4-requests 0 --naive-reps 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var', '$v', 'c5_tflops', round(d['c5_ingest']['tflops'],1), 'c3_req_s', round(d['c3_batch']['reordered']['requests_per_s'],1), 'naive_ms', round(d['naive_full_concat_p50_ttft_ms'],1), 'ttft', round(d['p50_ttft_ms'],3))"
done
