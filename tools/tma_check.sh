#!/usr/bin/env bash
# compute-sanitizer on the RF_KF_TMA variants: one small and one 640x480 case
mkdir -p gpurun_out
for v in ${VARIANTS:-tma tmaf}; do
  RF_LIB_PATH=$PWD/variants/lib_$v.so timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_volume_gpu.py -m gpu -q -x -k "script_golden or vga" > gpurun_out/san_$v.log 2>&1
  tail -30 gpurun_out/san_$v.log | head -40
done
