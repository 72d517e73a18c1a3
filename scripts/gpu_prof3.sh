#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expert_ffn or tile_widths" 2>&1 | tail -5
B="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
EXTRA=dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:ffn_layer2 -s 3 -c 1 -o gpurun_out/prof_dec128 $B > gpurun_out/ncu_dec.log 2>&1; echo "rc=$?"
README_FFN_NB=64 timeout 900 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:ffn_layer2 -s 3 -c 1 -o gpurun_out/prof_dec64 $B > gpurun_out/ncu_dec64.log 2>&1; echo "rc=$?"
ls gpurun_out
