#!/usr/bin/env bash
# The measurement set committed under profiles/ (one gpurun call):
#   GPU parity tests, the default bench line (N=1), the reference arm, the
#   ncu launch list of a 2-step bench, and one ncu --set full capture of the
#   fuse launches of tools/prof_workload.py (+ its algorithmic bytes).
# Usage: tools/round_profile.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/box_$TAG.txt
lscpu | grep -E "^CPU\(s\)|Model name" >> gpurun_out/box_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/benchref_$TAG.json 2> gpurun_out/benchref_$TAG.err
# the launch list of the timed steps only (NVTX range "timed" in bench.py)
timeout 1200 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 \
  --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv 2 > gpurun_out/launches_$TAG.json
timeout 300 python tools/prof_workload.py --build 20 --corrections 2 --json gpurun_out/workload_$TAG.json > /dev/null 2>&1
# the corrections' kernels after the 20 build integrations: the removal
# (k_check, k_fuse<kApplyRemove>) and the integration (k_fuse<kIntegrate>)
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "corrections/" -k regex:"k_fuse|k_check" \
  -o gpurun_out/prof_$TAG python tools/prof_workload.py --build 20 --corrections 2 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/prof_$TAG.ncu-rep gpurun_out/workload_$TAG.json gpurun_out/fuse_traffic_$TAG.json
cat gpurun_out/pytest_$TAG.log
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json')); r=d['roofline']
print('bench', round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline']['value'])"
