#!/bin/bash
# One ncu --set full capture of the config-2 expert FFN launch (ffn_layer2_kernel) and the launch list of the
# default bench command. Run under gpurun from the repo root; outputs land in gpurun_out/.
set -u
tag=${1:-cur}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_layer2 -s 2 -c 1 \
  -o gpurun_out/ffn_$tag -f python bench.py --steps 2 --warmup 3 --no-variants --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_$tag.log 2>&1
echo "ncu_full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-variants --no-e2e \
  --no-cpu-baseline > gpurun_out/launches_$tag.log 2>&1
echo "ncu_launches rc=$?"
