cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur21.so mb11=_variants/mb11.so --lams 4,5,3 --reps 7 2>&1 | tail -9
