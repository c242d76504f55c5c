#!/bin/bash
# Run commands against a TUNING build of the library (TKV_* environment knobs compiled in), then restore the release
# library: tools/tuning_run.sh "python tools/attn_trace_engine.py" ...
set -u
cp paper_2410_07590_b200/libtkv_b200.so /tmp/libtkv_release.so
make -s -C paper_2410_07590_b200 clean && make -s -j16 -C paper_2410_07590_b200 TUNING=1 > /dev/null 2>&1
for c in "$@"; do echo "== $c"; bash -c "$c"; done
cp /tmp/libtkv_release.so paper_2410_07590_b200/libtkv_b200.so
