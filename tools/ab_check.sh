#!/usr/bin/env bash
# A/B of the lean de-integration check (k_check, product build) against the
# k_fuse<kCheckRemove> pipeline (variants/lib_base.so, -DRF_LEAN_CHECK=0):
# parity tests on the product build, two rounds of the short bench per
# variant, and one ncu --set full capture of k_check.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_volume_gpu.py tests/test_edge_cases_gpu.py tests/test_reintegration.py tests/test_c2_replay_gpu.py tests/test_shard_failure_gpu.py tests/test_synth.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/abc_tests.log
cat gpurun_out/abc_tests.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/abc.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/abc.txt 2>&1
cat gpurun_out/abc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_check" -c 3 -o gpurun_out/prof_check python tools/prof_workload.py --build 20 --corrections 1 > /dev/null 2>&1
