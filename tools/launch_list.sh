#!/bin/bash
# ncu launch list (gpu__time_duration per kernel) of the C2 turbo step; $1 = engine flags, $2 = output tag
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$2.csv \
  python bench.py --steps 2 --warmup 3 --turbo-only --no-cpu-baseline --flags $1 > /dev/null 2>&1
python tools/step_breakdown.py gpurun_out/launches_$2.csv
