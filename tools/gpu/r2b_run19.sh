cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur2.so res2=_variants/res2.so maskend=_variants/maskend.so both=_variants/both2.so --lams 9,5,7 --reps 7 2>&1 | tail -15
