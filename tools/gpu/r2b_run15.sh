cd $GRAFT_REPO_ROOT
for v in new=paper_2404_18497_b200/libphobic_b200.so old=_variants/nok1big.so; do
  echo "== ${v%%=*}"; PHB_LIB=${v#*=} timeout 600 python tools/stage_perf_strings.py 2>&1 | tail -3
done
