cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur1.so a0=_variants/a0.so a50=_variants/a50.so a100=_variants/a100.so a200=_variants/a200.so --lams 9,5,7 --reps 7 2>&1 | tail -18
