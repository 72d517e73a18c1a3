#!/bin/bash
# Round evidence: all GPU tests, every bench config, ncu launch list + full-set captures of the hot kernels.
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-evidence}; mkdir -p gpurun_out/$TAG
O=gpurun_out/${TAG:-evidence}
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > $O/$name.log 2>&1; echo "$name rc=$?" | tee -a $O/summary.txt; }
rm -f $O/summary.txt
run tests 1500 python -m pytest tests -m gpu -q
tail -3 $O/tests.log
run smoke 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
tail -1 $O/smoke.log
run bench2 600 python bench.py --steps 30 --warmup 5
run bench1 300 python bench.py --config 1 --steps 50 --warmup 5
run bench3 600 python bench.py --config 3 --steps 30 --warmup 5
run bench4 900 python bench.py --config 4 --steps 5 --warmup 2
run bench4off 900 python bench.py --config 4 --offload --steps 3 --warmup 2
run bench5 900 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e
run benchref 600 python bench.py --impl reference --steps 5 --warmup 1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
run ncu_launch 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B
EXTRA=sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
run ncu_ffn 900 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:ffn_layer2 -s 2 -c 1 -o $O/prof_ffn $B
run ncu_perm 900 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:"route_cluster|move_rows_bulk" -s 2 -c 2 -o $O/prof_perm $B
B3="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
run ncu_dec 900 ncu --set full --metrics $EXTRA --clock-control none -k regex:ffn_layer2 -s 3 -c 1 -o $O/prof_dec $B3
cat $O/summary.txt
# (compute-sanitizer runs are closed on this GPU pool: earlier rounds' memcheck/synccheck logs are in profiles/)
