#!/usr/bin/env bash
mkdir -p gpurun_out
bash tools/ab_fp.sh
timeout 1500 python tools/bench_c4.py --reference --out gpurun_out/c4_r2f.json > gpurun_out/c4_r2f.log 2>&1
tail -2 gpurun_out/c4_r2f.log
timeout 1800 python tools/emulated_scaling.py > gpurun_out/scaling_r2.jsonl 2> gpurun_out/scaling_r2.err
tail -1 gpurun_out/scaling_r2.jsonl
