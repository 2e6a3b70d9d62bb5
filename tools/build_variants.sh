#!/bin/bash
# build feature variants of the library into _variants/<name>.so
set -e
cd "$(dirname "$0")/.."
mkdir -p _variants
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  PHB_NVCC_EXTRA="$flags" PHB_LIB=_variants/$name.so PHB_OBJ=_variants/obj_$name python -c "from paper_2404_18497_b200 import _build; _build.build()" > /dev/null
  echo built $name
done
