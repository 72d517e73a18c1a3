#!/bin/bash
# GPU iteration: build, GEMM parity, full gpu suite, bench, launch list + full ncu of the GEMMs.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > gpurun_out/$name.log 2>&1; echo "$name rc=$?" | tee -a gpurun_out/summary.txt; }
rm -f gpurun_out/summary.txt
run t_gemm 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expert_ffn or moe_layer or fused"
tail -c 2500 gpurun_out/t_gemm.log
run t_all 900 python -m pytest tests -m gpu -q
tail -c 1500 gpurun_out/t_all.log
run bench 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline
tail -c 3000 gpurun_out/bench.log
if [ "${PROF:-1}" = "1" ]; then
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
run launches 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B
EXTRA=sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
run ncu_gemm 900 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:"ffn_layer2|route_tile|finalize_dispatch" -s 3 -c 3 -o gpurun_out/prof_gemm $B
fi
