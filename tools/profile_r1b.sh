#!/bin/bash
set -u
B="python bench.py --steps 2 --warmup 3 --turbo-only --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_turbo2.csv $B > /dev/null 2>&1
for spec in "attn_tc:60:1" "gemm_tc:221:4" "attn_combine:40:1"; do
  IFS=: read -r k s c <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o gpurun_out/prof2_$k $B > gpurun_out/ncu2_$k.log 2>&1
  echo "$k rc=$?"
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --naive-reps 1 > gpurun_out/bench2.json 2>gpurun_out/bench2.err
