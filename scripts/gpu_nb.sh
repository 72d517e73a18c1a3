#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ep_gpu.py -m gpu -q -x 2>&1 | tail -15
for nb in 64 128; do
  README_FFN_NB=$nb timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b3_nb$nb.log 2>&1
  python - <<PY
import json
d=json.loads(open("gpurun_out/b3_nb$nb.log").readline())
print("nb=$nb", round(d["value"]), d["roofline"]["frac"], [(p["B"], round(p["hbm_frac"],3)) for p in d["decode_sweep"]])
u=d["unique_expert_sweep"]; print("  unique", [(p["unique_experts"], round(p["ms"]*1000,1)) for p in u["points"]], u["us_per_extra_expert"], u["intercept_us"])
PY
done
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b3.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b2.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/b2.log').readline()); print('c2', round(d['value']), d['roofline']['frac'], d['stage_ms_median'])
"
