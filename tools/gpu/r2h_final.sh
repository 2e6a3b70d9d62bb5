cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
tail -2 gpurun_out/r2h_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err
timeout 1500 bash tools/profile_r2h.sh > gpurun_out/r2h_profile.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2h_gpu_tests.log 2>&1
tail -3 gpurun_out/r2h_gpu_tests.log
