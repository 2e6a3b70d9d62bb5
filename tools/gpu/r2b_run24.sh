cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py pro4=_variants/pro4b.so pro2=_variants/pro2.so pro8=_variants/pro8.so --lams 9,5,4 --reps 7 2>&1 | tail -12
