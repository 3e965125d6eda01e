#!/usr/bin/env bash
# A/B including the end-to-end pass (host keyframes uploaded every step):
# the pair prefetches with an L2 evict_last priority (lib_pfel) vs base.
mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for r in 1 2; do
for lib in variants/lib_*.so; do
  tag=$(basename $lib .so)
  RF_LIB_PATH=$PWD/$lib timeout 400 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/abe_$tag.json 2>gpurun_out/abe_$tag.err
  python -c "
import json
d=json.load(open('gpurun_out/abe_$tag.json')); r=d['roofline']
print('$tag', round(d['value'],1), 'KF/s e2e', round(d['e2e']['value'],1), 'ms/step', round(d['ms_per_step'],2), 'int', round(r['avg_launch_us'],1), 'frac', round(r['frac'],3))
" || tail -3 gpurun_out/abe_$tag.err
done; done
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
