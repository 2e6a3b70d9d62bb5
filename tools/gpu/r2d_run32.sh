cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur8.so pu2=_variants/pu2.so nosat1=_variants/nosat1.so --lams 9,5,7 --reps 7 2>&1 | tail -12
