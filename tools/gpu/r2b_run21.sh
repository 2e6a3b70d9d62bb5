cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur3.so mbe1=_variants/mbe1.so mbe2=_variants/mbe2.so mbe8=_variants/mbe8.so --lams 4,5 --reps 7 2>&1 | tail -10
PHB_LIB=_variants/cur3.so timeout 600 python tools/stage_perf.py --lam 4 --enc ic-r --reps 3 2>&1 | tail -2
PHB_LIB=_variants/cur3.so timeout 600 python tools/stage_perf.py --lam 5 --enc ic-r --reps 3 2>&1 | tail -2
