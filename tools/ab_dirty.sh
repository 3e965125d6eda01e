#!/usr/bin/env bash
# A/B: new blocks on never-used slots skip the zero-fill (kDirtyFlag; the
# pool is cleared at creation) vs the committed build; parity tests first.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_volume_gpu.py tests/test_edge_cases_gpu.py tests/test_reintegration.py tests/test_c2_replay_gpu.py tests/test_pipeline_gpu.py tests/test_removal_failure_gpu.py tests/test_sharding_gpu.py tests/test_routing_gpu.py tests/test_shard_failure_gpu.py tests/test_mesh.py tests/test_fusion_gpu.py -m gpu -q 2>&1 | tail -5 > gpurun_out/abd_tests.log
cat gpurun_out/abd_tests.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/abd.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/abd.txt 2>&1
cat gpurun_out/abd.txt
