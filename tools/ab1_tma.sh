#!/usr/bin/env bash
# A/B of the k_fuse keyframe-tile TMA variant (variants/lib_tma.so, built with
# -DRF_KF_TMA=1 -DRF_FUSE_MINB=3) against the product build and a 3-CTA/SM
# build of it: parity tests on the variant, two rounds of the short bench,
# one ncu --set full capture of the fuse launches per variant.
mkdir -p gpurun_out
RF_LIB_PATH=$PWD/variants/lib_tma.so timeout 900 python -m pytest tests/test_volume_gpu.py tests/test_edge_cases_gpu.py tests/test_reintegration.py tests/test_c2_replay_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tma_tests.log
cat gpurun_out/tma_tests.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/ab1.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/ab1.txt 2>&1
cat gpurun_out/ab1.txt
for v in base tma; do
RF_LIB_PATH=$PWD/variants/lib_$v.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fuse" -s 20 -c 3 -o gpurun_out/prof_ab_$v python tools/prof_workload.py --build 20 --corrections 1 > /dev/null 2>&1
done
