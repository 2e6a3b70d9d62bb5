cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r2d_bench2.json 2> gpurun_out/r2d_bench2.err
tail -2 gpurun_out/r2d_bench2.err
