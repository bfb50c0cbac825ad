#!/bin/bash
# Build a variant of libfxg.so with extra -D flags for ONE source file, linked with
# the other objects of the normal build: tools/build_variant.sh <name> <file.cu> "<defs>"
# -> lib_alt/<name>/libfxg.so  (A/B of kernel tuning knobs with tools/kbench.py)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; defs=$3
out=lib_alt/$name; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2603_12016_b200/csrc --expt-relaxed-constexpr"
base=$(basename $src .cu)
nvcc $FL $defs -c paper_2603_12016_b200/csrc/$src -o $out/$base.o
objs=""
for o in paper_2603_12016_b200/build/*.o; do
  [ "$(basename $o)" = "$base.o" ] && continue; objs="$objs $o"; done
nvcc $ARCH -shared -cudart static -o $out/libfxg.so $out/$base.o $objs -lpthread -ldl -lrt
echo $out/libfxg.so
