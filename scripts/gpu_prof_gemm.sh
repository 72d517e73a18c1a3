#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
EXTRA=sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:ffn_gemm -s 2 -c 2 -o gpurun_out/prof_gemm2 $B > gpurun_out/ncu_gemm2.log 2>&1; echo "gemm rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $B > /dev/null 2>&1; echo "launch rc=$?"
