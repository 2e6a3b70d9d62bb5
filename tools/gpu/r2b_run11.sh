cd $GRAFT_REPO_ROOT
bash tools/query_variants.sh c32=paper_2404_18497_b200/libphobic_b200.so c32gt=_variants/encgt.so old=_variants/noqgt.so
