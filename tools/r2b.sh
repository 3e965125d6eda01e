#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_r2b.log
timeout 900 python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
bash tools/fusion_profile.sh r2b
tail -3 gpurun_out/pytest_r2b.log
python -c "
import json; d=json.load(open('gpurun_out/bench_r2b.json')); r=d['roofline']
print('bench', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), 'clocks', d['clocks'], d['config']['voxels_updated_per_integrate']['build_first3'])"
cat gpurun_out/fusion_r2b.json
