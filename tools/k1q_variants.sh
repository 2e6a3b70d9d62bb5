#!/bin/bash
# K1 (hash_count) and query timing of library variants: tools/k1q_variants.sh name=path ...
for v in "$@"; do
  name=${v%%=*}; path=${v#*=}
  echo "== $name"
  PHB_LIB=$path python tools/stage_perf.py --reps 3 2>&1 | grep "rep 2" | grep -o "hash_count=[0-9.]*ms"
  PHB_LIB=$path python tools/query_bench.py 100000000 ic-c 2>&1 | grep "ic-c matrix"
done
