#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b3.log 2> gpurun_out/b3.err
python -c "
import json
d=json.loads(open('gpurun_out/b3.log').readline())
print('c3', round(d['value']), round(d['roofline']['frac'],3), round(d['roofline']['step_frac'],3), d['stage_ms_mean'])
print([(p['B'], round(p['ms']*1000,1), round(p['hbm_frac'],3)) for p in d['decode_sweep']])
"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b2.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b2.log').readline()); print('c2', round(d['value']), round(d['roofline']['frac'],3), d['stage_ms_median'], d['clocks'])
"
timeout 600 python bench.py --config 4 --steps 3 --warmup 2 > gpurun_out/b4.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b4.log').readline()); print('c4', round(d['value']), round(d['roofline']['frac'],3), d['ms_per_step'], d['clocks'])
"
