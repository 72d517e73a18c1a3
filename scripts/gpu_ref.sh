#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1
timeout 300 python scripts/cublas_ref.py > gpurun_out/cublas_ref.json 2>&1; cat gpurun_out/cublas_ref.json
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench2.log 2>&1; tail -c 1500 gpurun_out/bench2.log
timeout 300 python scripts/cublas_ref.py > gpurun_out/cublas_ref2.json 2>&1; cat gpurun_out/cublas_ref2.json
