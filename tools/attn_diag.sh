#!/bin/bash
# Attention cost attribution on the GPU box: TUNING builds of deliberately invalid variants (ATTN_DIAG=1: no exp
# work, 2: no PV MMAs) traced in the C3 batch (tools/attn_trace_c3.py) beside the product kernel (0).
# Usage: bash tools/attn_diag.sh [variants...]   (default: 0 1 2); restores the release library.
set -u
P=paper_2410_07590_b200
cp $P/libtkv_b200.so /tmp/libtkv_release.so
for v in ${@:-0 1 2}; do
  make -s -C $P clean && make -s -j16 -C $P TUNING=1 XFLAGS="-DATTN_DIAG=$v" > /dev/null 2>&1
  echo "== ATTN_DIAG=$v"
  python tools/attn_trace_c3.py 2>&1 | grep -E -A9 "period|softmax S ready|kernel span|^tile"
done
make -s -C $P clean > /dev/null
cp /tmp/libtkv_release.so $P/libtkv_b200.so
