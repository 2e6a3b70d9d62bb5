cd $GRAFT_REPO_ROOT
timeout 900 python tools/variant_bench.py base=_variants/base.so e32=_variants/e32.so --lams 9,5,7,4 --reps 7 2>&1 | tail -10
PHB_LIB=_variants/e32.so timeout 1200 python -m pytest tests/test_gpu_api.py -q -x 2>&1 | tail -2
