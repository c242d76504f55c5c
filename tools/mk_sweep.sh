#!/bin/bash
# layer-kernel knob sweep on the C2 step (run under gpurun): builds a TUNING copy of the library, then restores.
# Arguments: env assignments per run, e.g.  "TKV_MK_L2_AHEAD=8" "TKV_MK_L2_AHEAD=8 TKV_MK_KROT=1"
set -u
cp paper_2410_07590_b200/libtkv_b200.so /tmp/libtkv_release.so
make -s -C paper_2410_07590_b200 clean && make -s -j16 -C paper_2410_07590_b200 TUNING=1 > /dev/null 2>&1
python tools/c2_step.py 0   # kernel chain
for cfg in "$@"; do env $cfg python tools/c2_step.py 128; done
[ -n "${MK_TRACE:-}" ] && env $MK_TRACE TKV_MK_TRACE=5 python tools/mk_trace.py
cp /tmp/libtkv_release.so paper_2410_07590_b200/libtkv_b200.so
