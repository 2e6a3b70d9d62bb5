cd $GRAFT_REPO_ROOT
for v in cs1=_variants/cs1.so cs2=_variants/cs2.so; do
  echo "== ${v%%=*}"
  PHB_LIB=${v#*=} timeout 600 python tools/stage_perf.py --lam 4 --enc ic-r --reps 3 2>&1 | tail -2
  PHB_LIB=${v#*=} timeout 600 python tools/stage_perf.py --lam 9 --enc ic-c --reps 3 2>&1 | tail -2
done
PHB_LIB=_variants/cs2.so timeout 1200 python -m pytest tests/test_gpu_api.py tests/test_gpu_distributed.py tests/test_gpu_query_encoded.py -q -x 2>&1 | tail -2
