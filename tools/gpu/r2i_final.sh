cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 bash tools/profile_r2i.sh > gpurun_out/r2i_profile.log 2>&1
python tools/ncu_to_json.py gpurun_out/r2i_search_c2.ncu-rep profiles/r2h_query_c2.ncu-rep > gpurun_out/r2i_ncu_to_json.log 2>&1
cp profiles/search_sm_c2.json profiles/search_traffic_c2.json profiles/query_c2.json gpurun_out/
timeout 900 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
tail -2 gpurun_out/r2i_bench.err
ncu -i gpurun_out/r2i_search_c2.ncu-rep --page details > gpurun_out/r2i_search_ncu_c2.txt 2>&1
