cd $GRAFT_REPO_ROOT
timeout 1200 python tools/variant_bench.py base=_variants/base.so ptr=_variants/ptr.so slim=_variants/slim.so both=_variants/both.so --lams 9,5,7 --reps 7 2>&1 | tail -15
