cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_query_encoded.py tests/test_gpu_compat.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c5 or strings" 2>&1 | tail -2
