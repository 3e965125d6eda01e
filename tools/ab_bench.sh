#!/usr/bin/env bash
# A/B the library variants in variants/: a short bench per variant.
for lib in variants/lib_*.so; do
  tag=$(basename $lib .so)
  RF_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/ab_$tag.json')); r=d['roofline']
print('$tag', round(d['value'],1), 'KF/s', 'fuse', round(r['avg_launch_us'],1), 'us', 'check share', round(r['check_ms_share'],3), 'fp share', round(r['footprint_ms_share'],3))
" || tail -3 gpurun_out/ab_$tag.err
done
