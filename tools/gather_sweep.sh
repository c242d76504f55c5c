#!/bin/bash
# A/B gather kernel variants (tools/libtkv_g<rows>_u<unroll>.so, built with -DGATHER_ROWS_CFG / -DGATHER_U_CFG)
# through the C2 step: p50 TTFT, KV-inject GB/s and its roofline fraction.
for so in "$@"; do
  TKV_LIB_PATH=$PWD/$so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --naive-reps 1 --c3-steps 0 --c4-requests 0 --c5-rounds 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', round(d['p50_ttft_ms'],3), round(d['kv_inject_gbs'],0), round(d['roofline']['frac'],3))"
done
