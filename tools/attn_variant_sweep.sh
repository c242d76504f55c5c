#!/bin/bash
# A/B attention ring variants (tools/libtkv_k<KST>v<VST>.so, -DATTN_KST / -DATTN_VST): C2 TTFT and attention
# utilisation, C3 batch req/s and batched attention utilisation.
for so in "$@"; do
  TKV_LIB_PATH=$PWD/$so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --naive-reps 1 --c3-steps 2 --c4-requests 0 --c5-rounds 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$so', round(d['p50_ttft_ms'],3), round(d['attention_roofline']['frac'],3), round(d['c3_batch']['reordered']['requests_per_s'],1), round(d['c3_batch']['attention_roofline']['frac'],3))"
done
