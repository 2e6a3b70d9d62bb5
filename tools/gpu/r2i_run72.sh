cd $GRAFT_REPO_ROOT
timeout 900 python tools/variant_bench.py base=_variants/base.so new=paper_2404_18497_b200/libphobic_b200.so --lams 9,5,7,4 --reps 7 2>&1 | tail -12
SAN=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $SAN --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/r2i_memcheck.log 2>&1; tail -2 gpurun_out/r2i_memcheck.log
timeout 2400 $SAN --tool racecheck --racecheck-report hazard python tools/sanitize_run.py > gpurun_out/r2i_racecheck.log 2>&1; tail -2 gpurun_out/r2i_racecheck.log
timeout 1800 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r2i_gpu_tests.log 2>&1
tail -2 gpurun_out/r2i_gpu_tests.log
