cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur13.so lateb=_variants/lateb.so --lams 9,5,7 --reps 7 2>&1 | tail -9
