#!/usr/bin/env bash
# A/B the library variants in variants/: the same short bench (identical step
# sequence) per variant; prints KF/s, ms/step and the event-timed per-launch
# averages of the fuse / check kernels.
for lib in variants/lib_*.so; do
  tag=$(basename $lib .so)
  RF_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/ab_$tag.json')); r=d['roofline']
rm=r.get('removal') or {}
print('$tag', round(d['value'],1), 'KF/s', round(d['ms_per_step'],2), 'ms/step ', r['kernel'], round(r['avg_launch_us'],1), 'us  frac', round(r['frac'],3), ' removal us/op', round(rm.get('us_per_op') or 0,1), ' shares fuse/check/fp', round(r['fuse_ms_share'],3), round(r['check_ms_share'],3), round(r['footprint_ms_share'],3))
" || tail -3 gpurun_out/ab_$tag.err
done
