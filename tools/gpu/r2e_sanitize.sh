cd $GRAFT_REPO_ROOT
SAN=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $SAN --tool memcheck --leak-check no python tools/sanitize_run.py > gpurun_out/r2e_memcheck.log 2>&1; tail -3 gpurun_out/r2e_memcheck.log
timeout 2400 $SAN --tool racecheck --racecheck-report hazard python tools/sanitize_run.py > gpurun_out/r2e_racecheck.log 2>&1; tail -3 gpurun_out/r2e_racecheck.log
timeout 1500 $SAN --tool synccheck python tools/sanitize_run.py > gpurun_out/r2e_synccheck.log 2>&1; tail -3 gpurun_out/r2e_synccheck.log
