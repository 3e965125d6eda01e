#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 2400 python tools/bench_c3_slice.py > gpurun_out/c3_slice.json 2> gpurun_out/c3_slice.err
tail -3 gpurun_out/c3_slice.err; cat gpurun_out/c3_slice.json
timeout 2400 python tools/emulated_scaling.py --voxel 0.004 --modes replicated --shards 1,2,4,8 > gpurun_out/scaling_4mm_r2.jsonl 2> gpurun_out/scaling_4mm_r2.err
tail -2 gpurun_out/scaling_4mm_r2.err; tail -1 gpurun_out/scaling_4mm_r2.jsonl
