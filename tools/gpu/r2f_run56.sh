cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_api.py -q -x -k "long_and_mixed" 2>&1 | tail -3
