cd $GRAFT_REPO_ROOT
timeout 900 python tools/variant_bench.py base=_variants/base.so l64=_variants/l64.so l64w96=_variants/l64w96.so --lams 9,5,7 --reps 5 2>&1 | tail -12
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
for v in l64; do
  echo "== $v"
  PHB_LIB=_variants/$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:k_search -s 1 -c 1 --csv python tools/run_build.py --n 100000000 --reps 2 2>/dev/null | grep k_search | awk -F'","' '{print $(NF-2), $NF}'
done
PHB_LIB=_variants/l64.so timeout 1200 python -m pytest tests/test_gpu_api.py -q -x 2>&1 | tail -2
