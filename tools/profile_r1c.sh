#!/bin/bash
# ncu launch list + --set full captures of the top kernels for the C2 turbo path (under gpurun).
set -u
B="python bench.py --steps 2 --warmup 3 --turbo-only --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_turbo.csv $B > /dev/null 2>&1
python tools/step_breakdown.py gpurun_out/launches_turbo.csv > gpurun_out/step_breakdown.txt
for spec in "attn_tc:60:1" "gemm_tc:221:4" "gather_rope:3:1"; do
  IFS=: read -r k s c <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
