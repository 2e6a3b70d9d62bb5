cd $GRAFT_REPO_ROOT
timeout 1200 python tools/variant_bench.py cur=paper_2404_18497_b200/libphobic_b200.so w88=_variants/w88.so w80=_variants/w80.so w80b=_variants/w80b.so --lams 9,5,7 --reps 7 2>&1 | tail -14
