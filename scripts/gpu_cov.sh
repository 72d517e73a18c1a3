#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_ep_gpu.py -m gpu -q 2>&1 | tail -15
timeout 300 python bench.py --config 1 --steps 50 --warmup 5 > gpurun_out/bench1.log 2>&1; tail -c 800 gpurun_out/bench1.log
timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench5.log 2>&1; tail -c 1500 gpurun_out/bench5.log
