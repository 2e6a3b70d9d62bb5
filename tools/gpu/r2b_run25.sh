cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur5.so pf=_variants/pf.so --lams 9,5,4 --reps 7 2>&1 | tail -9
