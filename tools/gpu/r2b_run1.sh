cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_stages.py -x -q -k "cta" 2>&1 | tail -5
timeout 1200 python tools/variant_bench.py base=_variants/base.so cta=paper_2404_18497_b200/libphobic_b200.so acc128=_variants/acc128.so nosat4=_variants/nosat4.so both=_variants/both.so --lams 9,5 --reps 5 2>&1 | tail -30
timeout 600 python tools/stage_perf.py --reps 3 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_api.py -x -q 2>&1 | tail -5
