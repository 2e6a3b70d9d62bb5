cd $GRAFT_REPO_ROOT
bash tools/query_variants.sh cur=paper_2404_18497_b200/libphobic_b200.so qcarve=_variants/qcarve.so qtabg=_variants/qtabg.so qtabgc=_variants/qtabgc.so
timeout 900 python tools/variant_bench.py old=_variants/base.so cur=paper_2404_18497_b200/libphobic_b200.so --lams 9,5 --reps 7 2>&1 | tail -6
