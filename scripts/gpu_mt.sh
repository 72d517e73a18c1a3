#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2410_19123_b200.build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile_widths or tile_edges or teacher or config3 or moe_layer_end" 2>&1 | tail -3
BENCH_ARGS="--config 3 --steps 30 --warmup 5" bash scripts/gpu_ab.sh README_FFN_MT=256 | tail -4
