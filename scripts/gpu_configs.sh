#!/bin/bash
# All GPU parity tests + the bench for configs 2, 3, 4 (and the oracle reference arm).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > gpurun_out/$name.log 2>&1; echo "$name rc=$?" | tee -a gpurun_out/summary.txt; }
rm -f gpurun_out/summary.txt
run t_all 1200 python -m pytest tests -m gpu -q
tail -c 2500 gpurun_out/t_all.log
#run bench2 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline
tail -c 3000 gpurun_out/bench2.log
run bench3 600 python bench.py --config 3 --steps 30 --warmup 5
#run bench2e 600 python bench.py --steps 30 --warmup 5 --eager --no-cpu-baseline --no-e2e
tail -c 1500 gpurun_out/bench2e.log
tail -c 4000 gpurun_out/bench3.log
#run bench4 900 python bench.py --config 4 --steps 5 --warmup 2
tail -c 2000 gpurun_out/bench4.log
#run benchref 600 python bench.py --impl reference --steps 5 --warmup 1
tail -c 1500 gpurun_out/benchref.log
