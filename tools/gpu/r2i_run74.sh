cd $GRAFT_REPO_ROOT
timeout 900 python tools/variant_bench.py base=_variants/base.so h8=_variants/h8.so --lams 9,7,5,4 --reps 7 2>&1 | tail -12
PHB_LIB=_variants/h8.so timeout 1200 python -m pytest tests/test_gpu_api.py tests/test_gpu_stages.py -q -x 2>&1 | tail -2
