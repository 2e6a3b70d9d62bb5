cd $GRAFT_REPO_ROOT
for l in 4 5; do PHB_LIB=_variants/stats.so timeout 600 python tools/search_stats.py 20000000 $l 2>&1 | tail -20; done
