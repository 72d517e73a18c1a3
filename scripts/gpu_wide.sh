#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expert_ffn or tile_widths or moe_layer" 2>&1 | tail -2
for w in 1 0 1; do
  README_FFN_WIDE=$w timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b2_w$w.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/b2_w$w.log').readline()); print('wide=$w', round(d['value']), round(d['roofline']['frac'],3), d['stage_ms_median'], d['clocks'])
"
done
