cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py old=_variants/base.so cur=paper_2404_18497_b200/libphobic_b200.so fdpair=_variants/fdpair.so t32=_variants/t32.so slim=_variants/slim.so all3=_variants/all3.so --lams 9,5 --reps 5 2>&1 | tail -16
bash tools/query_variants.sh cur=paper_2404_18497_b200/libphobic_b200.so qna=_variants/qna.so qgtna=_variants/qgtna.so
