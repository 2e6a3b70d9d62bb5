cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur19.so nomask=_variants/nomask.so --lams 9,5,7,4 --reps 7 2>&1 | tail -11
PHB_LIB=_variants/nomask.so timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_api.py -q -x 2>&1 | tail -2
