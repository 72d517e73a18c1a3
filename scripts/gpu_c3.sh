#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "router" 2>&1 | tail -3 | tee gpurun_out/rtest.log
timeout 300 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b3.log 2> gpurun_out/b3.err
tail -3 gpurun_out/b3.err
python scripts/show_b3.py gpurun_out/b3.log
