#!/bin/bash
# Round profile of the C2 turbo step (run under gpurun; one GPU). $1 = tag (e.g. r2a). Outputs: gpurun_out/.
#  1. launch list (gpu__time_duration per kernel, --clock-control none) -> per-class share of one step
#  2. ncu --set full of the hot kernels: gather, attention (+ combine), one layer's 4 projection GEMMs, the
#     epilogue kernels -> DRAM bytes per launch (roofline.traffic) and the key metrics
set -u
T=${1:-r2}
# --flags 256 = TKV_FLAG_NO_GRAPHS: under ncu a graph-replayed gate/up GEMM node of the bench fails to launch
# ("LaunchFailed", grid 0,0,0; r2p) although the same graphs profile fine from tools/c2_step.py and the bench is
# memcheck-clean; ncu serializes every launch anyway, so the kernels and their durations are those of the graph path
B="python bench.py --steps 2 --warmup 3 --turbo-only --no-cpu-baseline --flags 256"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > /dev/null 2>&1
python tools/step_breakdown.py gpurun_out/${T}_launches.csv gpurun_out/${T}_launch_share.json > gpurun_out/${T}_launches_summary.txt
# launch indices inside the first measured turbo step: skip the warm-up steps' kernels
for spec in "gather_rope:3:1" "attn_tc_kernel:121:1" "attn_tc_combine:94:1" "gemm_tc:485:4" "residual_kernel:242:2" "qkv_epilogue:122:1"; do
  IFS=: read -r k s c <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c -o gpurun_out/${T}_full_$k $B > gpurun_out/${T}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
