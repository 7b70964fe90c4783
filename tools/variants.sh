#!/bin/bash
# Diagnostic build variants of the library (compile-time knobs), selected at run time
# with ALAYA_LIB_VARIANT=<name>:  tools/variants.sh name "-DKNOB=1 ..." [name "-D..."]...
set -e
cd "$(dirname "$0")/../paper_2504_10326_b200/csrc"
while [ $# -ge 2 ]; do
  mkdir -p ../variants/$1
  make -j16 OUT=../variants/$1/libalaya_b200.so BUILD=/tmp/alaya_build_var_$1 EXTRA="$2" > /dev/null
  echo "built variant $1 ($2)"
  shift 2
done
