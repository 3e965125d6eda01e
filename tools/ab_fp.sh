#!/usr/bin/env bash
# A/B: footprint tiles beyond the first wave handed to the first CTAs that
# finish (dynamic) vs a static stride; parity tests on the product build.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_volume_gpu.py tests/test_c2_replay_gpu.py tests/test_pipeline_gpu.py tests/test_sharding_gpu.py tests/test_routing_gpu.py tests/test_edge_cases_gpu.py -m gpu -q 2>&1 | tail -3 > gpurun_out/abf_tests.log
cat gpurun_out/abf_tests.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/abf.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/abf.txt 2>&1
cat gpurun_out/abf.txt
