#!/bin/bash
# Experiment builds: recompile one source with extra nvcc flags and link it
# with the cached objects of the default build into
# paper_2409_14222_b200/_variants/libvanka_<tag>.so (select with VK_LIB=...).
#   tools/build_variant.sh <tag> <source.cu> [nvcc flags...]
set -e
tag=$1; src=$2; shift 2
cd "$(dirname "$0")/.."
B=paper_2409_14222_b200/_build
V=paper_2409_14222_b200/_variants
mkdir -p $V/$tag
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr \
  $ARCH "$@" -c paper_2409_14222_b200/csrc/$src -o $V/$tag/${src%.cu}.o
objs=""
for o in $B/*.o; do
  b=$(basename $o)
  if [ "$b" = "${src%.cu}.o" ]; then objs="$objs $V/$tag/$b"; else objs="$objs $o"; fi
done
nvcc $ARCH -shared -o $V/libvanka_$tag.so $objs -lcudart
echo $V/libvanka_$tag.so
