#!/bin/bash
# compute-sanitizer over the kernel-level tests and one small engine path (run under gpurun).
# memcheck: out-of-bounds / misaligned global + shared accesses; racecheck: shared-memory hazards (mbarrier and
# TMA/UMMA traffic is asynchronous-proxy and outside its model); synccheck: illegal barrier use.
# Summary lines -> gpurun_out/sanitize_summary.txt ($1 = tag)
set -u
T=${1:-r2}
OUT=gpurun_out/${T}_sanitize_summary.txt
: > $OUT
TESTS="tests/test_gpu_kernels.py tests/test_gpu_parity.py::test_four_paths_vs_golden"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 --error-exitcode 99 \
    python -m pytest -q -x -m gpu $TESTS -p no:cacheprovider > gpurun_out/${T}_sanitize_$tool.log 2>&1
  rc=$?
  echo "== $tool rc=$rc" >> $OUT
  grep -E "ERROR SUMMARY|passed|failed|error" gpurun_out/${T}_sanitize_$tool.log | tail -5 >> $OUT
done
cat $OUT
