cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur25.so ll8=_variants/ll8.so ll10=_variants/ll10.so --lams 6,7,9 --reps 7 2>&1 | tail -12
