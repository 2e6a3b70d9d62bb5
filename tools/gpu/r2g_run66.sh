cd $GRAFT_REPO_ROOT
for v in cs1=_variants/cs1.so cs3=_variants/cs3.so; do
  echo "== ${v%%=*}"
  PHB_LIB=${v#*=} timeout 600 python tools/stage_perf.py --lam 4 --enc ic-r --reps 3 2>&1 | tail -2 | head -1
  PHB_LIB=${v#*=} timeout 600 python tools/stage_perf.py --lam 9 --enc ic-c --reps 3 2>&1 | tail -2 | head -1
done
PHB_LIB=_variants/cs3.so timeout 1200 python -m pytest tests/test_gpu_api.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -2
