#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pipeline" 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b2.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b2.log').readline()); print('c2', round(d['value']), d['e2e'])
"
