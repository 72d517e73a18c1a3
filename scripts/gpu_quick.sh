#!/bin/bash
# Quick GPU iteration: build, GEMM parity (both kernels), full gpu suite, bench.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > gpurun_out/$name.log 2>&1; echo "$name rc=$?" | tee -a gpurun_out/summary.txt; }
rm -f gpurun_out/summary.txt
run t_gemm 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expert_ffn"
tail -c 2500 gpurun_out/t_gemm.log
run t_all 900 python -m pytest tests -m gpu -q
tail -c 1500 gpurun_out/t_all.log
run bench 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline
tail -c 3000 gpurun_out/bench.log
README_FFN_KERNEL=1cta run bench1cta 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
tail -c 800 gpurun_out/bench1cta.log
