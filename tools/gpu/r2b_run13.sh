cd $GRAFT_REPO_ROOT
for v in cur=paper_2404_18497_b200/libphobic_b200.so k3m3=_variants/k3m3.so k3m4=_variants/k3m4.so k3n4m4=_variants/k3n4m4.so k3n16=_variants/k3n16.so; do
  echo "== ${v%%=*}"; PHB_LIB=${v#*=} python tools/scatter_micro.py 2>&1 | tail -1
done
