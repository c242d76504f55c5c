#!/bin/bash
# In-chain timeline (tools/timeline.py) of library variants on one box: each paper_2410_07590_b200/libtkv_<v>.so is
# copied over the product library in turn; the product library is restored at the end.
# Usage: bash tools/timeline_variants.sh <variant>...   (e.g. after make XFLAGS=... && cp libtkv_b200.so libtkv_x.so)
P=paper_2410_07590_b200
cp $P/libtkv_b200.so /tmp/libtkv_keep.so
for v in "$@"; do
  cp $P/libtkv_$v.so $P/libtkv_b200.so
  echo "== $v"
  python tools/timeline.py 2>&1 | grep -E "gap (epilogue|attention)->|epilogue us|attention us|p50"
done
cp /tmp/libtkv_keep.so $P/libtkv_b200.so
