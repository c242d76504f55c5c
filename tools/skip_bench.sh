#!/bin/bash
# Cost attribution of the C2 turbo step: p50 with kernel classes dropped (TKV_TIMING_SKIP bitmask; results
# numerically invalid), through the TUNING build (make TUNING=1 BUILD=.../build_tuning LIB=.../libtkv_tuning.so).
# 1 = residual after O-proj, 2 = residual after down-proj, 4 = qkv epilogue, 8 = attention
export TKV_LIB_PATH=${TKV_LIB_PATH:-paper_2410_07590_b200/libtkv_tuning.so}
for m in "$@"; do
  echo -n "skip $m: "; TKV_TIMING_SKIP=$m timeout 300 python tools/c2_step.py 2>/dev/null | tail -1
done
