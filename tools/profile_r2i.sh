#!/bin/bash
# Round-2 (final, u32 sweep entries) measurement artifacts (run under gpurun; writes gpurun_out/):
#   r2i_search_c2.ncu-rep    ncu --set full of k_search at C2 (100M keys, lambda=9)
#   r2i_build_metrics.csv    dram bytes / time / issue of every kernel of one C2 build
#   r2i_launches_c2.csv      launch list (gpu__time_duration) of a short bench run
set -x
ncu --set full --clock-control none --import-source on -k regex:k_search -s 1 -c 1 \
    -o gpurun_out/r2i_search_c2 python tools/run_build.py --n 100000000 --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none -s 12 -c 14 --csv --log-file gpurun_out/r2i_build_metrics.csv \
    python tools/run_build.py --n 100000000 --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2i_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-configs --no-c3 --no-cpu-baseline \
    > gpurun_out/r2i_launches_bench.log 2>&1
