#!/usr/bin/env bash
# A/B runs of bench.py under different environments (same step sequence).
# Usage: tools/ab_env.sh "tag1:VAR=val VAR2=val" "tag2:..." ...
# A throw-away short run first absorbs first-launch effects on a fresh box.
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for spec in "$@"; do
  tag=${spec%%:*}
  envs=${spec#*:}
  env $envs timeout 300 python bench.py --steps ${STEPS:-6} --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "
import json
d=json.load(open('gpurun_out/ab_$tag.json')); r=d['roofline']
print('$tag', round(d['value'],1), 'KF/s', round(d['ms_per_step'],2), 'ms/step  fuse', round(r['avg_launch_us'],1), 'us  frac', round(r['frac'],3), ' shares fuse/check/fp', round(r['fuse_ms_share'],3), round(r['check_ms_share'],3), round(r['footprint_ms_share'],3))
" || tail -3 gpurun_out/ab_$tag.err
done
