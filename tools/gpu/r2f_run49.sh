cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur17.so g8=_variants/g8.so --lams 9,5,7 --reps 7 2>&1 | tail -9
