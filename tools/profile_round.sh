#!/bin/bash
# Round profile of the C2 turbo path (run under gpurun, one GPU). Outputs in gpurun_out/ (scratch); copy the
# summaries into profiles/ with tools/ncu_collect.py.
#   1. launch list (gpu__time_duration per kernel, --clock-control none) of the bench command itself
#   2. one `ncu --set full` capture per hot kernel (gather+RoPE, attention, combine, GEMM instances)
set -u
TAG=${1:-r1}
B="python bench.py --steps 2 --warmup 3 --turbo-only --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > /dev/null 2>&1
python tools/step_breakdown.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches_summary.txt
# kernel:skip:count  (skip counts launches of that kernel before the capture; step 1 of 5 starts after warm-up)
for spec in "gather_rope:3:1" "attn_tc_kernel:90:1" "attn_tc_combine:90:1" "gemm_tc_kernel:360:4"; do
  IFS=: read -r k s c <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c \
    -o gpurun_out/${TAG}_full_$k $B > gpurun_out/${TAG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
# large-M (8256-token full-concat prefill) gate/up + down GEMMs: the tensor-bound tiling
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 2 \
  -o gpurun_out/${TAG}_full_gemm_bigM python tools/naive_once.py > gpurun_out/${TAG}_ncu_gemm_bigM.log 2>&1
echo "gemm_bigM rc=$?"
