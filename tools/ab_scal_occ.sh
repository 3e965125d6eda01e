#!/usr/bin/env bash
# Does a higher-occupancy fuse kernel (fewer registers, spills) help the small
# per-shard launches of the 8-shard emulation?  G = 1 and 8, replicated.
mkdir -p gpurun_out
for tag in base minb6; do
  RF_LIB_PATH=$PWD/variants/lib_$tag.so timeout 1500 python tools/emulated_scaling.py --shards 1,8 --modes replicated > gpurun_out/scal_$tag.jsonl 2> gpurun_out/scal_$tag.err
  python -c "
import json
for line in open('gpurun_out/scal_$tag.jsonl'):
    d=json.loads(line)
    if 'summary' in d: print('$tag', d); continue
    sd=d['shards_detail']
    print('$tag', d['mode'], d['shards'], 'wall', d['max_shard_ms_per_step'], 'fuse', round(max(s['fuse'] for s in sd),3), 'check', round(max(s['check'] for s in sd),3))
"
done
