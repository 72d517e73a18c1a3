#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expert_ffn or moe_layer or fused or gate_up or stack" 2>&1 | tail -3
for v in 0; do README_LAB=$v timeout 300 python scripts/gemm_lab.py; done 2>&1 | tee gpurun_out/lab.log
README_FFN_KERNEL=split timeout 300 python scripts/gemm_lab.py 2>&1 | tee -a gpurun_out/lab.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench2.log 2>&1; tail -c 1500 gpurun_out/bench2.log
