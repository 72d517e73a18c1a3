#!/bin/bash
# Full GPU suite + smoke + default bench line.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/tests
O=gpurun_out/tests
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > $O/$name.log 2>&1; echo "$name rc=$?" | tee -a $O/summary.txt; }
rm -f $O/summary.txt
run t_all 1500 python -m pytest tests -m gpu -q
tail -c 1500 $O/t_all.log
run smoke 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
tail -1 $O/smoke.log
run bench 600 python bench.py ${BENCH_ARGS:---steps 30 --warmup 5}
grep '^{' $O/bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('stage_ms_median'), d['roofline']['frac'], d.get('e2e',{}).get('value'))"
cat $O/summary.txt
