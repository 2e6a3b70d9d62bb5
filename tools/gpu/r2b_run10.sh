cd $GRAFT_REPO_ROOT
bash tools/query_variants.sh new=paper_2404_18497_b200/libphobic_b200.so old=_variants/noqgt.so
timeout 600 python -m pytest tests/test_gpu_query_encoded.py tests/test_gpu_api.py -q -x 2>&1 | tail -2
