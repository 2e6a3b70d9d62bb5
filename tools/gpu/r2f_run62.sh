cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur24.so mbe1=_variants/mbe1.so mbe05=_variants/mbe05.so mbe4=_variants/mbe4.so --lams 4,5,3 --reps 7 2>&1 | tail -15
