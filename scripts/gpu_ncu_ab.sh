#!/bin/bash
# DRAM bytes / duration of the config-2 FFN launch under ncu, default vs env overrides given as arguments.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/ncuab
O=gpurun_out/ncuab
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
B="python bench.py ${BENCH_ARGS:---steps 2 --warmup 1} --no-cpu-baseline --no-e2e --no-variants"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,gpc__cycles_elapsed.max.per_second
i=0
for kv in "DEFAULT=1" "$@"; do
  env $kv timeout 600 ncu --metrics $M --clock-control none -k regex:${KREGEX:-ffn_layer2} -s ${SKIP:-2} -c ${COUNT:-3} --csv $B > $O/n$i.csv 2>$O/n$i.err
  echo "== $kv"; python - $O/n$i.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
rows = rows[[i for i, r in enumerate(rows) if r and r[0] == "ID"][0]:]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
for r in rows[1:]:
    print("  ", r[ki][:40], r[mi], r[vi], r[ui])
PY
  i=$((i+1))
done
