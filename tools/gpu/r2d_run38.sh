cd $GRAFT_REPO_ROOT
for v in q2c=_variants/q2c.so q1=_variants/q1.so; do echo "== ${v%%=*}"; PHB_LIB=${v#*=} timeout 600 python tools/query_bench_strings.py 2>&1 | tail -2; done
