# C5 / C3 in-chain timelines (tools/timeline.py) of library variants: bash tools/c5c3_variants.sh <variant>...
P=paper_2410_07590_b200
cp $P/libtkv_b200.so /tmp/keep.so
for v in "$@"; do cp $P/libtkv_$v.so $P/libtkv_b200.so; echo "== $v"; TL_C5=1 TL_GAPS=0 python tools/timeline.py 2>&1 | tail -2; TL_C3=1 TL_GAPS=0 python tools/timeline.py 2>&1 | grep -E "epilogue us|p50"; done
cp /tmp/keep.so $P/libtkv_b200.so
