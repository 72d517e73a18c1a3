#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2410_19123_b200.build > /dev/null 2>&1 || { python -m paper_2410_19123_b200.build 2>&1 | tail -20; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split_k or tile_widths or tile_edges or teacher or fuzz or config3" 2>&1 | tail -15
python scripts/ffn_lab.py README_FFN_SPLITK=2,1 64 256 512 1024
BENCH_ARGS="--config 3 --steps 30 --warmup 5" bash scripts/gpu_ab.sh README_FFN_SPLITK=1 | tail -4
