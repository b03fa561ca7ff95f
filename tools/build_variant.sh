#!/bin/bash
# Build a variant of the library with extra nvcc defines for one source:
#   tools/build_variant.sh NAME SOURCE.cu -DFOO=1 ...   -> _variants/libNAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p _variants/$name
objs=""
for o in paper_2408_07436_b200/build/*.o; do
  b=$(basename $o .o)
  if [ "$b.cu" == "$src" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include "$@" \
      -c -o _variants/$name/$b.o paper_2408_07436_b200/csrc/$src
    objs="$objs _variants/$name/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/lib$name.so $objs
echo _variants/lib$name.so
