#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "offloaded" 2>&1 | tail -25
timeout 900 python bench.py --config 4 --offload --steps 3 --warmup 2 > gpurun_out/bench_offload.log 2> gpurun_out/bench_offload.err
echo "bench exit $?"; tail -3 gpurun_out/bench_offload.err; cut -c1-3000 gpurun_out/bench_offload.log
