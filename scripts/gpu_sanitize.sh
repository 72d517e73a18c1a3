#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for k in "route_bit_exact" "dispatch or combine" "tile_edges and merged" "moe_layer_end_to_end and fused" "router_step" "offloaded_stack"; do
  echo "=== $k"
  timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$k" > gpurun_out/san.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|Invalid|passed|failed" gpurun_out/san.log | head -5
done
