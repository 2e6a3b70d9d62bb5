cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur16.so pfn=_variants/pfn.so --lams 9,5,4 --reps 7 2>&1 | tail -9
