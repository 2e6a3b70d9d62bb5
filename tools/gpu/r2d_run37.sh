cd $GRAFT_REPO_ROOT
for v in q2=_variants/q2.so q1=_variants/q1.so; do echo "== ${v%%=*}"; PHB_LIB=${v#*=} timeout 600 python tools/query_bench_strings.py 2>&1 | tail -2; done
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_query_encoded.py -q -x -k "string or strings or str_keys or corpus" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c5 or strings" 2>&1 | tail -2
