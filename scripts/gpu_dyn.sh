#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2410_19123_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile_widths or tile_edges" 2>&1 | tail -2
README_FFN_DYNAMIC=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "expert_ffn or moe_layer or stack" 2>&1 | tail -2
