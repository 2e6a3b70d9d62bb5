cd $GRAFT_REPO_ROOT
for v in new=paper_2404_18497_b200/libphobic_b200.so old=_variants/nostaged.so; do
  echo "== ${v%%=*}"; PHB_LIB=${v#*=} timeout 600 python tools/stage_perf_strings.py 2>&1 | tail -2
done
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_api.py -q -x -k "murmur or string or strings or corpus or str_keys" 2>&1 | tail -2
