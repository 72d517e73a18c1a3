#!/bin/bash
# Functional check of the N>1 bench path with 4 and 8 ranks sharing one GPU (gloo; numbers meaningless).
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2410_19123_b200.build > /dev/null 2>&1 || exit 1
for n in 4 8; do
for ep in peer nccl; do
README_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) bench.py --gpus $n --steps 2 --warmup 3 --tokens 1024 --ep $ep 2>&1 | grep '^{' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('n=$n ep=$ep', d['config'].get('ep_exchange'), d['config'].get('ep_fallback'), round(d['ms_per_step'],2), d.get('step_mode'), 'e2e', (d.get('e2e') or {}).get('ms_per_step'))
"
done; done
