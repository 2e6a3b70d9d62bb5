cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
for v in base pad nc4; do
  echo "== $v"
  PHB_LIB=_variants/$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:k_search -s 1 -c 1 --csv python tools/run_build.py --n 100000000 --reps 2 2>/dev/null | grep k_search | awk -F'","' '{print $(NF-2), $NF}'
done
