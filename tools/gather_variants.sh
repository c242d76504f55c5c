#!/bin/bash
# C2 / C3 in-chain gather (tools/timeline.py) of library variants: bash tools/gather_variants.sh <variant>...
P=paper_2410_07590_b200
cp $P/libtkv_b200.so /tmp/libtkv_keep.so
for v in "$@"; do
  cp $P/libtkv_$v.so $P/libtkv_b200.so
  echo "== $v"
  python tools/timeline.py 2>&1 | grep -E "p50" | sed 's/| gemm us.*//'
  TL_C3=1 TL_GAPS=0 python tools/timeline.py 2>&1 | grep -E "p50" | sed 's/| gemm us.*//'
done
cp /tmp/libtkv_keep.so $P/libtkv_b200.so
