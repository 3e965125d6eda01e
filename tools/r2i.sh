#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_r2i.log
cat gpurun_out/pytest_r2i.log
timeout 900 python bench.py > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err
tail -2 gpurun_out/bench_r2i.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r2i.json')); r=d['roofline']
print('bench', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3), 'e2e', round(d['e2e']['value'],1), d['e2e']['clocks'])"
STEPS=8 bash tools/ab_bench.sh > gpurun_out/abg.txt 2>&1
STEPS=8 bash tools/ab_bench.sh >> gpurun_out/abg.txt 2>&1
cat gpurun_out/abg.txt
timeout 1500 python tools/bench_c3_slice.py > gpurun_out/c3_slice.json 2> gpurun_out/c3_slice.err
cat gpurun_out/c3_slice.json
