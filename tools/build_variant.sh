#!/bin/bash
# Build a variant of the product library with extra nvcc defines into build/variants/<name>/.
# usage: tools/build_variant.sh <name> [-DFOO=1 ...] [--sparse-from <git-rev>]
set -e
name=$1; shift
defs=()
rev=""
while [ $# -gt 0 ]; do
  case "$1" in
    --sparse-from) rev=$2; shift 2;;
    *) defs+=("$1"); shift;;
  esac
done
out=build/variants/$name
mkdir -p $out/obj
src=paper_1403_1649_b200/csrc
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -ccbin /usr/bin/g++ -Xcompiler -fPIC,-O2"
objs=()
for f in $src/*.cu; do
  b=$(basename $f .cu)
  if [ "$b" = "sparse" ] && [ -n "$rev" ]; then
    git show $rev:$f > $out/sparse_$rev.cu
    (cd $src && $NV "${defs[@]}" -I. -c ../../$out/sparse_$rev.cu -o ../../$out/obj/$b.o) &
  else
    $NV "${defs[@]}" -c $f -o $out/obj/$b.o &
  fi
  objs+=($out/obj/$b.o)
done
for f in $src/*.cpp; do
  b=$(basename $f .cpp)
  /usr/bin/g++ -std=c++17 -O2 -fPIC -I/usr/local/cuda/include -c $f -o $out/obj/$b.cpp.o &
  objs+=($out/obj/$b.cpp.o)
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libaggmg_b200.so "${objs[@]}" -Xcompiler -fPIC
echo built $out/libaggmg_b200.so
