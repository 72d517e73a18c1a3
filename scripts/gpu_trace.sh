#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/trace
O=gpurun_out/trace
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
python scripts/trace_lab.py > $O/trace_graph.txt 2>&1; echo rc=$?
TRACE_GRAPH=0 python scripts/trace_lab.py > $O/trace_eager.txt 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/trace/trace_graph.txt", "gpurun_out/trace/trace_eager.txt"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e, open(f).read()[-2000:]); continue
    print(f)
    for r in d["us_from_route_start"]:
        print("  ", {k: round(v, 1) for k, v in r.items()})
PY
