#!/usr/bin/env bash
# One gpurun call: GPU parity tests, a short bench, optionally the ncu launch
# list of a 2-step bench (LAUNCHES=1) and an ncu --set full capture of the
# fuse kernels on the fixed profiling workload (NCU=1).  Usage: tools/gpu_check.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_$TAG.log
  cat gpurun_out/pytest_$TAG.log
fi
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:---no-e2e} \
  > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
python - "$TAG" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
r = d["roofline"]
print(f"value {d['value']:.1f} KF/s  ms/corr {d['ms_per_step']:.2f}  fuse avg {r['avg_launch_us']:.1f} us "
      f"frac {r['frac']:.3f}  shares fuse {r['fuse_ms_share']:.2f} check {r['check_ms_share']:.2f} "
      f"fp {r['footprint_ms_share']:.2f}  e2e {(d.get('e2e') or {}).get('value')}")
PY
if [ "${LAUNCHES:-1}" = "1" ]; then
  timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_$TAG.csv 2 > gpurun_out/launches_$TAG.json
  python - "$TAG" <<'PY'
import json, sys
l = json.load(open(f"gpurun_out/launches_{sys.argv[1]}.json"))
print("launch list: total_us/2 steps", round(l["total_us"], 1))
for k, v in list(l["kernels"].items())[:8]:
    print(f"  {k:40s} n={v['count']:4d} avg={v['avg_us']:8.2f} share={v['share']:.3f}")
PY
fi
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_fuse}" -s ${NCU_S:-20} -c ${NCU_C:-3} \
    -o gpurun_out/prof_$TAG python tools/prof_workload.py --build 20 --corrections 1 > /dev/null 2>&1
fi
