#!/bin/bash
# All GPU parity tests + the bench for every config (and the oracle reference arm).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
run() { local name=$1; shift; local t=$1; shift; timeout $t "$@" > gpurun_out/$name.log 2>&1; echo "$name rc=$?" | tee -a gpurun_out/summary.txt; }
rm -f gpurun_out/summary.txt
TESTS=0; [ "${TESTS:-1}" = "1" ] && run t_all 1200 python -m pytest tests -m gpu -q && tail -c 600 gpurun_out/t_all.log
run bench2 600 python bench.py --steps 30 --warmup 5
run bench1 300 python bench.py --config 1 --steps 50 --warmup 5
run bench3 600 python bench.py --config 3 --steps 30 --warmup 5
run bench4 900 python bench.py --config 4 --steps 5 --warmup 2
run bench5 900 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e
run benchref 600 python bench.py --impl reference --steps 5 --warmup 1
for f in bench2 bench1 bench3 bench4 bench5 benchref; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    l = [x for x in open(f"gpurun_out/{f}.log") if x.startswith("{")][-1]
    d = json.loads(l)
    print(f, "value=%.4g" % d["value"], "ms=%.4g" % d["ms_per_step"], "frac=", (d.get("roofline") or {}).get("frac"),
          "stages=", d.get("stage_ms_median"), "router=", d.get("router"), "clocks=", d.get("clocks"))
except Exception as e:
    print(f, "ERR", e)
PY
done
