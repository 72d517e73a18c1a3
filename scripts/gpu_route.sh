#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "route or moe_layer or stack" 2>&1 | tail -2
for rt in 256 64 32; do
  README_ROUTE_TILE=$rt timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b2_rt$rt.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/b2_rt$rt.log').readline()); print('rt=$rt', round(d['value']), d['ms_per_step'], d['stage_ms_median'])
"
done
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b3.log 2>&1
python scripts/show_b3.py gpurun_out/b3.log
