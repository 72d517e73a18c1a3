#!/bin/bash
# config-2 timeline (trace_lab) under env overrides given as arguments
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/trace
python -m paper_2410_19123_b200.build > /dev/null 2>&1 || exit 1
for kv in "DEFAULT=1" "$@"; do
  env $kv TRACE_T=${TRACE_T:-8192} python scripts/trace_lab.py > gpurun_out/trace/t.txt 2>&1
  python - "$kv" <<'PY'
import json, sys
d = json.load(open("gpurun_out/trace/t.txt"))
rs = d["us_from_route_start"][1:]
keys = ["route_end", "dispatch_start", "dispatch_end", "ffn_past_prologue", "ffn_first_tile_ready", "ffn_end", "event_us"]
print(sys.argv[1], {k: round(sum(r[k] for r in rs) / len(rs), 1) for k in keys})
PY
done
