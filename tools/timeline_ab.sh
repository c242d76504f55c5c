# Same-box A/B of library variants through the in-chain timeline: bash tools/timeline_ab.sh <variant>... (C2, then C3)
P=paper_2410_07590_b200
for round in 1 2; do
  for v in "$@"; do
    echo -n "$v C2: "; TKV_LIB_PATH=$P/libtkv_$v.so TL_GAPS=0 timeout 300 python tools/timeline.py 2>&1 | tail -1
  done
done
for v in "$@"; do
  echo -n "$v C3: "; TKV_LIB_PATH=$P/libtkv_$v.so TL_C3=1 TL_GAPS=0 timeout 600 python tools/timeline.py 2>&1 | tail -2 | tr '\n' ' '; echo
done
