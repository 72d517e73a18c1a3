#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for tool in racecheck synccheck; do
for k in "route_bit_exact" "router_step or router_forward" "dispatch_rmsnorm or combine_weighted" "tile_edges and merged"; do
  echo "=== $tool $k"
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$k" > gpurun_out/san.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Barrier|passed|failed" gpurun_out/san.log | head -5
done
done
