#!/usr/bin/env bash
# compute-sanitizer over the round-2 device paths: k_check and the removal
# failure paths, the synth renderer, sharded marching cubes (peer tables),
# cross-shard verdicts (k_shard_sync), the eval grid index, fusion.
mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
{
echo "== memcheck: removal failure, synth, sharded mesh, eval, fusion"
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_removal_failure_gpu.py tests/test_synth.py tests/test_mesh_sharded_gpu.py \
  tests/test_eval_gpu.py tests/test_fusion_gpu.py tests/test_staged_uploads_gpu.py -m gpu -q -x \
  -k "not vga and not corridor_many" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|error" | tail -5
echo "== memcheck: shard failure (k_shard_sync), G=2"
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_shard_failure_gpu.py -m gpu -q -x -k "2-False or (2 and False)" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|error" | tail -5
echo "== racecheck: removal failure + sharded mesh"
timeout 1500 compute-sanitizer --tool racecheck --target-processes all --print-limit 20 \
  python -m pytest tests/test_removal_failure_gpu.py tests/test_mesh_sharded_gpu.py tests/test_staged_uploads_gpu.py -m gpu -q -x 2>&1 | grep -E "passed|failed|RACECHECK SUMMARY|hazard" | tail -5
} > gpurun_out/sanitize_r2.txt 2>&1
cat gpurun_out/sanitize_r2.txt
