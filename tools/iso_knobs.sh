cp paper_2410_07590_b200/libtkv_b200.so /tmp/libtkv_release.so
make -s -C paper_2410_07590_b200 clean && make -s -j16 -C paper_2410_07590_b200 TUNING=1 > /dev/null 2>&1
for k in "" "8,200,1,1" "4,110,1,1" "4,110,2,1"; do echo "== knobs $k"; TKV_GEMM_KNOBS=$k python tools/gemm_iso.py; done
cp /tmp/libtkv_release.so paper_2410_07590_b200/libtkv_b200.so
