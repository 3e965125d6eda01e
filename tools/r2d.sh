#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_shard_failure_gpu.py tests/test_removal_failure_gpu.py -m gpu -q 2>&1 | tail -5 > gpurun_out/sf_r2d.log
timeout 900 python -m pytest tests/test_shard_failure_gpu.py -m gpu -q 2>&1 | tail -3 >> gpurun_out/sf_r2d.log
cat gpurun_out/sf_r2d.log
bash tools/ab_rev.sh
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2d.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r2d.csv 2 > gpurun_out/launches_r2d.json
head -c 600 gpurun_out/launches_r2d.json
