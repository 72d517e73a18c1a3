#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2410_19123_b200.build > /dev/null 2>&1 || exit 1
for rep in 1 2 3; do
for kv in "X=1" "README_PERM_UNROLL_D=8 README_PERM_UNROLL_C=8"; do
env $kv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-variants 2>&1 | grep "^{" | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$kv', round(d['hbm']['dispatch_frac'],3), round(d['hbm']['combine_frac'],3))"
done; done
