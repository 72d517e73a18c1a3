#!/bin/bash
# Cluster route + gather dispatch with per-row flags: parity, then A/B bench against the lookback path.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r2
O=gpurun_out/r2
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > $O/$name.log 2>&1; echo "$name rc=$?" | tee -a $O/summary.txt; }
rm -f $O/summary.txt
run t_route 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "route"
tail -c 1500 $O/t_route.log
run t_layer 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "moe_layer or fused or graph or config2 or equivariance or host_pipeline"
tail -c 1500 $O/t_layer.log
run bench_new 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
README_ROUTE=lookback run bench_old 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
run launches 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B
run t_all 1200 python -m pytest tests -m gpu -q
tail -c 1500 $O/t_all.log
cat $O/summary.txt
