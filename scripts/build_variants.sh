#!/bin/bash
# Builds library variants into paper_2204_00525_b200/lib_<name>/ with extra
# -D flags: scripts/build_variants.sh name1 "flags1" name2 "flags2" ...
set -e
cd "$(dirname "$0")/../paper_2204_00525_b200/csrc"
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  make -j 8 LIBDIR=lib_$name EXTRA="$flags" > /tmp/build_$name.log 2>&1 || { tail -20 /tmp/build_$name.log; exit 1; }
  echo "built lib_$name ($flags)"
done
