cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur11.so g25=_variants/g25.so g50=_variants/g50.so g200=_variants/g200.so --lams 9,5,7 --reps 7 2>&1 | tail -15
