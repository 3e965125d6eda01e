#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_shard_failure_gpu.py -m gpu -q -x 2>&1 | tail -60 > gpurun_out/sf_lean.log
RF_LIB_PATH=$PWD/variants/lib_base.so timeout 600 python -m pytest tests/test_shard_failure_gpu.py -m gpu -q 2>&1 | tail -5 > gpurun_out/sf_base.log
timeout 900 python -m pytest tests/test_synth.py tests/test_mesh_sharded_gpu.py tests/test_mesh.py -m gpu -q 2>&1 | tail -40 > gpurun_out/new_tests.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/abc2.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/abc2.txt 2>&1
cat gpurun_out/abc2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_check" -c 3 -o gpurun_out/prof_check2 python tools/prof_workload.py --build 20 --corrections 1 > /dev/null 2>&1
tail -3 gpurun_out/sf_lean.log; cat gpurun_out/sf_base.log; tail -3 gpurun_out/new_tests.log
