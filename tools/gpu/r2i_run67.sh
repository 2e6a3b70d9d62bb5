cd $GRAFT_REPO_ROOT
timeout 900 python tools/variant_bench.py base=_variants/base.so nc4=_variants/nc4.so nc4_88=_variants/nc4_88.so nc2=_variants/nc2.so --lams 9,5,7 --reps 5 2>&1 | tail -16
PHB_LIB=_variants/nc4.so timeout 1200 python -m pytest tests/test_gpu_api.py -q -x 2>&1 | tail -2
