cd $GRAFT_REPO_ROOT
for v in nopro=_variants/cur4.so pro4=paper_2404_18497_b200/libphobic_b200.so nopro=_variants/cur4.so pro4=paper_2404_18497_b200/libphobic_b200.so; do
  echo "== ${v%%=*}"; PHB_LIB=${v#*=} timeout 600 python tools/stage_perf.py --n 1000000000 --reps 3 2>&1 | tail -3
done
