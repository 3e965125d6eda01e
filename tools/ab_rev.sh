#!/usr/bin/env bash
# A/B of the fuse kernels' walk direction over the touched list (L2 reuse of
# the preceding op's last blocks; RF_FUSE_REVERSE bit 0 integrate, bit 1
# removal) + an ncu capture of the correction footprints (k_footprint).
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/abr.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/abr.txt 2>&1
cat gpurun_out/abr.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_footprint" -s 20 -c 4 \
  -o gpurun_out/prof_fp python tools/prof_workload.py --build 20 --corrections 2 > /dev/null 2>&1
