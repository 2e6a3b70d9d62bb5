cd $GRAFT_REPO_ROOT
timeout 600 python tools/e2e_timeline.py 2>&1 | tail -60
