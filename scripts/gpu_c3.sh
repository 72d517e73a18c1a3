#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b3.log 2> gpurun_out/b3.err
tail -3 gpurun_out/b3.err
python -c "
import json
d=json.loads(open('gpurun_out/b3.log').readline())
print(round(d['value']), d['roofline'], d['stage_ms_mean'], d['e2e'], d['clocks'])
print([(p['B'], round(p['ms']*1000,1), round(p['hbm_frac'],3)) for p in d['decode_sweep']])
"
