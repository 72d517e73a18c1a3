#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/b2h.log 2> gpurun_out/b2h.err
tail -3 gpurun_out/b2h.err
python -c "
import json
d=json.loads(open('gpurun_out/b2h.log').readline()); print(round(d['value']), round(d['roofline']['frac'],3), d['hbm'])
"
