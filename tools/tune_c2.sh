#!/bin/bash
# C2 turbo-step A/B of tuning knobs (run under gpurun): builds a TUNING copy of the library (TKV_* environment knobs
# compiled in), times tools/c2_step.py once per argument (env assignments, e.g. "TKV_GEMM_KNOBS=4,110,1,1"), restores
# the release library. Results are for choosing defaults only; bench.py refuses a TUNING build.
set -u
cp paper_2410_07590_b200/libtkv_b200.so /tmp/libtkv_release.so
make -s -C paper_2410_07590_b200 clean && make -s -j16 -C paper_2410_07590_b200 TUNING=1 > /dev/null 2>&1
FLAGS=${FLAGS:-0}
python tools/c2_step.py $FLAGS
for cfg in "$@"; do env $cfg python tools/c2_step.py $FLAGS; done
cp /tmp/libtkv_release.so paper_2410_07590_b200/libtkv_b200.so
