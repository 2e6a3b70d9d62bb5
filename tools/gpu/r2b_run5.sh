cd $GRAFT_REPO_ROOT
for f in 1 0.5 0.25 0.125 0.0625; do
  echo "== PHB_FUSE_SPLIT=$f"
  PHB_FUSE_SPLIT=$f timeout 600 python tools/variant_bench.py cur=paper_2404_18497_b200/libphobic_b200.so --lams 9,5 --reps 7 2>&1 | grep lambda= | head -2
done
timeout 1500 python -m pytest tests/test_gpu_api.py tests/test_gpu_stages.py -x -q 2>&1 | tail -3
