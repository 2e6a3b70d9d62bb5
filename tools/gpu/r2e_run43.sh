cd $GRAFT_REPO_ROOT
for v in cur=_variants/cur14.so hpre=_variants/hpre.so; do
  echo "== ${v%%=*}"; PHB_LIB=${v#*=} timeout 600 python tools/stage_perf_strings.py 2>&1 | tail -2
  PHB_LIB=${v#*=} timeout 600 python tools/query_bench_strings.py 2>&1 | tail -1
done
PHB_LIB=_variants/hpre.so timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_api.py -q -x -k "murmur or string or strings or str_keys or corpus" 2>&1 | tail -2
