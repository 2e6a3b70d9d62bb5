cd $GRAFT_REPO_ROOT
for tr in p2p nccl; do
  timeout 900 python bench.py --gpus 2 --same-device --backend gloo --transport $tr --keys 20000000 --steps 3 --warmup 3 --e2e-steps 1 --no-configs --no-cpu-baseline > gpurun_out/r2f_multigpu_2rank_same_device_$tr.json 2> gpurun_out/r2f_multigpu_$tr.err
  tail -2 gpurun_out/r2f_multigpu_$tr.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hash_pairs|k_query32s" -s 2 -c 2 -o gpurun_out/r2f_query_strings python tools/query_bench_strings.py > /dev/null 2>&1
cd /tmp && python $GRAFT_REPO_ROOT/tools/ncu_summary.py $GRAFT_REPO_ROOT/gpurun_out/r2f_query_strings.ncu-rep 15 > $GRAFT_REPO_ROOT/gpurun_out/r2f_query_strings_ncu.txt 2>&1
