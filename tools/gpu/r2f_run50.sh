cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur18.so k4m6=_variants/k4m6.so k4m4=_variants/k4m4.so --lams 9,5,7 --reps 7 2>&1 | tail -12
