# A/B of library variants on one box: each variant is copied over the product library (bench.py refuses
# TKV_LIB_PATH), then the C2 + C3 bench sample runs. Usage: bash tools/variant_ab.sh <tag> <variant>...
set -u
export PYTHONUNBUFFERED=1
tag=$1; shift
P=paper_2410_07590_b200
cp $P/libtkv_b200.so $P/libtkv_default.so
if [ "${RUN_TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_gputest.log
fi
timeout 120 python tools/attn_trace.py > gpurun_out/${tag}_tr_iso.txt 2>&1
TKV_LIB_PATH=$P/libtkv_tuning.so TKV_TRACE_LAYER=14 timeout 200 python tools/attn_trace_engine.py > gpurun_out/${tag}_tr_c2.txt 2>&1
for v in "$@"; do
  cp $P/libtkv_$v.so $P/libtkv_b200.so
  timeout 120 python tools/attn_trace.py > gpurun_out/${tag}_tr_iso_$v.txt 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --c5-rounds 0 --c4-requests 0 ${BENCH_ARGS:-} > gpurun_out/${tag}_ab_$v.json 2> gpurun_out/${tag}_ab_$v.err
  echo "bench $v rc=$?"
  python - gpurun_out/${tag}_ab_$v.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c3 = d.get("c3_batch", {})
print(f"  C2 {d['ms_per_step']:.3f} ms  attn {d['attention_roofline']['device_ms_per_request']:.3f} ms ({d['attention_roofline']['frac']:.3f})"
      f"  C3 {c3.get('reordered', {}).get('requests_per_s', 0):.1f} req/s attn frac {c3.get('attention_roofline', {}).get('frac', 0):.3f}"
      f"  naive {d.get('naive_full_concat_p50_ttft_ms', 0):.1f} ms")
PY
done
cp $P/libtkv_default.so $P/libtkv_b200.so
