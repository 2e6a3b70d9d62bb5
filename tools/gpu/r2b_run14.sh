cd $GRAFT_REPO_ROOT
for v in cur=paper_2404_18497_b200/libphobic_b200.so cs2=_variants/cs2.so cs8=_variants/cs8.so cs32=_variants/cs32.so; do
  echo "== ${v%%=*}"; PHB_LIB=${v#*=} python tools/scatter_micro.py 2>&1 | tail -1
done
