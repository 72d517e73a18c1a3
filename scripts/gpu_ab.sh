#!/bin/bash
# A/B: default path vs env overrides given as arguments (each "NAME=VAL" runs one extra bench)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/ab
O=gpurun_out/ab
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
rm -f $O/ab.txt
show() { grep '^{' $1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$2', round(d['value']/1e6,3), 'step', round(d['ms_per_step'],4), d.get('stage_ms_median'), d['roofline'].get('frac'), d['roofline'].get('step_frac'), d['clocks']['sm_mhz'])" >> $O/ab.txt; }
for rep in 1 2; do
timeout 300 python bench.py ${BENCH_ARGS:---steps 30 --warmup 5} --no-cpu-baseline --no-e2e > $O/b_default.log 2>&1; show $O/b_default.log default
for kv in "$@"; do env $kv timeout 300 python bench.py ${BENCH_ARGS:---steps 30 --warmup 5} --no-cpu-baseline --no-e2e > $O/b_x.log 2>&1; show $O/b_x.log "$kv"; done
done
cat $O/ab.txt
