#!/bin/bash
# One gpurun call: GPU parity tests in stages (each under its own timeout), smoke, a short bench.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > gpurun_out/$name.log 2>&1; echo "$name rc=$?" | tee -a gpurun_out/summary.txt; }
rm -f gpurun_out/summary.txt
run t_route 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "route or dispatch or combine or build_experts"
run t_f32 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "f32"
run t_gemm 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bf16_teacher"
run t_rest 600 python -m pytest tests -m gpu -q -k "not route and not dispatch and not combine and not build_experts and not f32 and not bf16_teacher"
run smoke 300 python __graft_entry__.py smoke
run bench 900 python bench.py --steps 10 --warmup 3
tail -c 3000 gpurun_out/t_gemm.log
cat gpurun_out/summary.txt
