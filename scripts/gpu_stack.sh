#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/stack
O=gpurun_out/stack
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "stack or moe_layer" > $O/t.log 2>&1; echo "tests rc=$?"; tail -2 $O/t.log
show() { grep '^{' $1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$2', round(d['value']/1e3,2), 'Ktok/s', round(d['ms_per_step'],3), 'ms', d['roofline']['frac'], d['clocks']['sm_mhz'])"; }
timeout 900 python bench.py --config 4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $O/b4_new.log 2>&1; show $O/b4_new.log gather
README_DISPATCH=scatter timeout 900 python bench.py --config 4 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $O/b4_old.log 2>&1; show $O/b4_old.log scatter
