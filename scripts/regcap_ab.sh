#!/bin/bash
# Lab A/B (measurement only): the default build (FFN uncapped, scatter dispatch) against a build whose FFN is
# capped at $1 registers and whose gather dispatch CTA has $2 threads, so the two kernels can be co-resident
# (gather forms, PDL). Same box, sequential. Run under gpurun from the repo root; results in gpurun_out/.
set -u
cap=${1:-192}; thr=${2:-256}
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build --force > /dev/null 2>&1
for r in 1 2; do
  timeout 300 python bench.py --no-variants --no-e2e --no-cpu-baseline > gpurun_out/regcap_default_$r.jsonl 2>/dev/null
done
README_NVCC_EXTRA="-DREADME_FFN_MAXREG=$cap -DREADME_GATHER_THREADS=$thr" python -m paper_2410_19123_b200.build --force --verbose > gpurun_out/regcap_build.log 2>&1
for r in 1 2; do
  for v in scatter gather fused; do
    README_DISPATCH=$v timeout 300 python bench.py --no-variants --no-e2e --no-cpu-baseline > gpurun_out/regcap_${v}_$r.jsonl 2>/dev/null
  done
done
README_DISPATCH=gather timeout 120 python scripts/trace_lab.py > gpurun_out/regcap_trace_gather.json 2>&1
python -m paper_2410_19123_b200.build --force > /dev/null 2>&1   # leave the default library behind
