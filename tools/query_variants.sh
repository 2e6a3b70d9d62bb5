#!/bin/bash
# query rate of library variants: tools/query_variants.sh name=path ...
for v in "$@"; do
  name=${v%%=*}; path=${v#*=}
  echo "== $name"
  PHB_LIB=$path python tools/query_bench.py 100000000 ic-c 2>&1 | grep -v Warn | grep -v from_numpy
done
