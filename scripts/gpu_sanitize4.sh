#!/bin/bash
# compute-sanitizer over the decode variant (128-row m-tiles, 8-stage ring) and the shape fuzz.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/san
O=gpurun_out/san
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
run() { local tool=$1; shift; local k=$1; shift
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$k" > $O/san.log 2>&1
  echo "$tool | $k | rc=$? | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $O/san.log | tr '\n' ' ' | cut -c1-200)"; }
run memcheck "fuzz"
run memcheck "tile_widths or tile_edges or config3"
run synccheck "tile_widths"
