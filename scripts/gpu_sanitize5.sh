#!/bin/bash
# compute-sanitizer over the FFN with the second CTA's A-load skip (tiles of <= 64 rows): decode-sized
# tiles, the tile-width A/B matrix and the shape fuzz.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/san
O=gpurun_out/san
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
run() { local tool=$1; shift; local k=$1; shift
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$k" > $O/san.log 2>&1
  echo "$tool | $k | rc=$? | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $O/san.log | tr '\n' ' ' | cut -c1-200)"; }
run memcheck "tile_widths_bitwise_equal"
run memcheck "fuzz_bf16"
run synccheck "tile_widths_bitwise_equal and 40"
run racecheck "tile_widths_bitwise_equal and 40"
