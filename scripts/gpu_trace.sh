#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/trace
O=gpurun_out/trace
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
for T in ${TRACE_TS:-8192}; do
TRACE_T=$T python scripts/trace_lab.py > $O/trace_graph_$T.txt 2>&1; echo rc=$?
TRACE_T=$T README_DISPATCH=scatter python scripts/trace_lab.py > $O/trace_scatter_$T.txt 2>&1
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/trace/trace_*_*.txt")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", open(f).read()[-1500:]); continue
    print(f)
    for r in d["us_from_route_start"][1:4]:
        print("  ", {k: round(v, 1) for k, v in r.items()})
PY
