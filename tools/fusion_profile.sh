#!/usr/bin/env bash
# Keyframe-fusion evidence: the fusion bench line, the ncu
# launch list of its kernels (2 keyframes = 10 frames) and one ncu --set full
# capture of every fusion kernel class of one frame + one fuse_color.
# Usage: tools/fusion_profile.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python tools/bench_fusion.py > gpurun_out/fusion_$TAG.json 2> gpurun_out/fusion_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/fusion_launches_$TAG.csv python tools/bench_fusion.py --keyframes 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_dw_warp|k_merge|k_scatter|k_fuse_color|k_gauss|k_blur|k_pairwise|Scan" -s 40 -c 16 \
  -o gpurun_out/prof_fusion_$TAG python tools/bench_fusion.py --keyframes 2 > /dev/null 2>&1
