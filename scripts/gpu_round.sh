#!/bin/bash
# Round evidence under gpurun: the whole GPU suite, smoke(), and bench lines for configs 2 (default) and 3.
# Usage: bash scripts/gpu_round.sh TAG [extra bench configs...]; outputs in gpurun_out/.
set -u
tag=${1:-cur}; shift || true
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$tag.log
timeout 600 python bench.py > gpurun_out/bench2_$tag.jsonl 2> gpurun_out/bench2_$tag.err
echo "bench2 rc=$?"
for c in "$@"; do
  timeout 900 python bench.py --config $c > gpurun_out/bench${c}_$tag.jsonl 2> gpurun_out/bench${c}_$tag.err
  echo "bench$c rc=$?"
done
