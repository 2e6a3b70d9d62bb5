cd $GRAFT_REPO_ROOT
timeout 900 python tools/variant_bench.py base=_variants/base.so pad=_variants/pad.so pad400=_variants/pad400.so nc4=_variants/nc4.so --lams 9,5 --reps 5 2>&1 | tail -10
