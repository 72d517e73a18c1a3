#!/bin/bash
# compute-sanitizer over the kernels added in r01 v12+: cluster route, gather dispatch with row flags,
# FFN waiting on row flags, gather pre-norm dispatch.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/san
O=gpurun_out/san
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
run() { local tool=$1; shift; local k=$1; shift
  timeout 1200 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$k" > $O/san.log 2>&1
  echo "$tool | $k | rc=$? | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $O/san.log | tr '\n' ' ' | cut -c1-200)"; }
run memcheck "route_bit_exact and cluster"
run memcheck "route_large_batch"
run memcheck "moe_layer_end_to_end and (fused or gather or scatter)"
run memcheck "moe_stack_end_to_end"
run racecheck "route_bit_exact and cluster"
run synccheck "route_bit_exact and cluster"
run racecheck "moe_layer_end_to_end and gather and bf16"
