#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/rlab
O=gpurun_out/rlab
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
rm -f $O/lab.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "route" > $O/t_route.log 2>&1; echo "t_route rc=$?"; tail -2 $O/t_route.log
README_ROUTE=lookback python scripts/route_lab.py >> $O/lab.txt 2>&1
python scripts/route_lab.py >> $O/lab.txt 2>&1
for c in 4 8 16; do README_ROUTE=cluster README_ROUTE_CLUSTER=$c python scripts/route_lab.py >> $O/lab.txt 2>&1; done
cat $O/lab.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench.log 2>&1; echo "bench rc=$?"
grep '^{' $O/bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stage_ms_median'])"
