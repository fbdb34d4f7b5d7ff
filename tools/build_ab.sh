#!/bin/bash
# Build the library with one source file swapped, for side-by-side timing:
#   tools/build_ab.sh <name> <file.cu to substitute> -> build/ab/libotn_<name>.so
# (use with OTN_LIB_AB=build/ab/libotn_<name>.so)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; sub=$2
tmp=$ROOT/paper_2504_02067_b200/csrc_ab_$name
rm -rf "$tmp"; mkdir -p "$tmp" "$ROOT/build/ab"
cp "$ROOT"/paper_2504_02067_b200/csrc/*.cu "$ROOT"/paper_2504_02067_b200/csrc/*.cuh \
   "$ROOT"/paper_2504_02067_b200/csrc/*.h "$tmp"/
cp "$sub" "$tmp/$(basename "${3:-otn_cg.cu}")"
cd "$tmp"
srcs=$(ls *.cu | sed 's/\.cu$//')
for f in $srcs; do
  nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a \
       -c $f.cu -o $f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$ROOT/build/ab/libotn_$name.so" \
     $(for f in $srcs; do echo $f.o; done) -lcudart_static
cd "$ROOT"; rm -rf "$tmp"
echo "built build/ab/libotn_$name.so"
