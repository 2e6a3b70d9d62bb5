cd $GRAFT_REPO_ROOT
bash tools/query_variants.sh cur=paper_2404_18497_b200/libphobic_b200.so qpf=_variants/qpf.so qpf_nk2=_variants/qpf8.so
