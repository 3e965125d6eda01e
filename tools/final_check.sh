#!/usr/bin/env bash
# Final verification of the committed tree: GPU tests, smoke(), a short bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_final.log
cat gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 8 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json')); r=d['roofline']
print('bench', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],3), 'step_frac', round(r['step_frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
