cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur0.so g1e025=_variants/g1e025.so g1e05=_variants/g1e05.so g1e1=_variants/g1e1.so g1e2=_variants/g1e2.so --lams 9,5,7 --reps 7 2>&1 | tail -18
