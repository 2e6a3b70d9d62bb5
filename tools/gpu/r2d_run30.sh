cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur6.so w8=_variants/w8.so nosat2=_variants/nosat2.so --lams 9,5,7 --reps 7 2>&1 | tail -12
