#!/usr/bin/env bash
# A/B: k_gc with four independent nz loads per thread vs one
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_volume_gpu.py tests/test_c2_replay_gpu.py tests/test_removal_failure_gpu.py tests/test_sharding_gpu.py tests/test_reintegration.py -m gpu -q 2>&1 | tail -3 > gpurun_out/abg_tests.log
cat gpurun_out/abg_tests.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/abg.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/abg.txt 2>&1
cat gpurun_out/abg.txt
