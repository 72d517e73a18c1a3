#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/ncudec
O=gpurun_out/ncudec
python -m paper_2410_19123_b200.build > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
B3="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
M=gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,gpc__cycles_elapsed.max,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:ffn_layer2 -s 3 -c 2 --csv $B3 > $O/dec.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ffn_layer2 -s 3 -c 1 -o $O/dec_full $B3 > $O/dec_full.log 2>&1
echo done
