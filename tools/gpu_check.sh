#!/usr/bin/env bash
# One gpurun call: GPU parity tests, a short bench, and an ncu capture of the
# fuse kernels on the fixed profiling workload.  Usage: tools/gpu_check.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_$TAG.log
cat gpurun_out/pytest_$TAG.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
python - "$TAG" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
r = d["roofline"]
print(f"value {d['value']:.1f} KF/s  ms/corr {d['ms_per_step']:.2f}  fuse avg {r['avg_launch_us']:.1f} us "
      f"frac {r['frac']:.3f}  shares fuse {r['fuse_ms_share']:.2f} check {r['check_ms_share']:.2f} "
      f"fp {r['footprint_ms_share']:.2f}")
PY
if [ "${NCU:-1}" = "1" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_fuse}" -s ${NCU_S:-20} -c ${NCU_C:-3} \
    -o gpurun_out/prof_$TAG python tools/prof_workload.py --build 20 --corrections 1 > /dev/null 2>&1
fi
