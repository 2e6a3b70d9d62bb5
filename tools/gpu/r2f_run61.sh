cd $GRAFT_REPO_ROOT
timeout 1500 python tools/variant_bench.py cur=_variants/cur23.so mb16=_variants/mb16.so --lams 4,5,3 --reps 7 2>&1 | tail -9
PHB_LIB=_variants/mb16.so timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_api.py -q -x 2>&1 | tail -2
