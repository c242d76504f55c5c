#!/bin/bash
# ncu captures for the C2 turbo path (run under gpurun). Outputs land in gpurun_out/.
set -u
B="python bench.py --steps 2 --warmup 3 --turbo-only --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_turbo.csv $B > /dev/null 2>&1
for spec in "attn_tc:60:1" "gemm_tc:221:4" "residual_norm:300:1" "swiglu:150:1" "qkv_epilogue:100:1" "attn_combine:40:1" "gather_rope:3:1"; do
  IFS=: read -r k s c <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
