cd $GRAFT_REPO_ROOT
timeout 600 python tools/query_bench_strings.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_query32_bytes -s 1 -c 1 -o gpurun_out/r2d_query_bytes python tools/query_bench_strings.py > /dev/null 2>&1
cd /tmp && python $GRAFT_REPO_ROOT/tools/ncu_summary.py $GRAFT_REPO_ROOT/gpurun_out/r2d_query_bytes.ncu-rep 20
