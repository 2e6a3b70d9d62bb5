cd $GRAFT_REPO_ROOT
PHB_LIB=_variants/stats.so timeout 600 python tools/search_stats.py 20000000 9 2>&1 | tail -20
