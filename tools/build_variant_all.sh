#!/bin/bash
# Whole-library variant: every .cu compiled with extra -D flags (knobs shared by
# several translation units, e.g. the S0 tile): tools/build_variant_all.sh <name> "<defs>"
set -e
cd "$(dirname "$0")/.."
name=$1; defs=$2
out=lib_alt/$name; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2603_12016_b200/csrc --expt-relaxed-constexpr"
for f in paper_2603_12016_b200/csrc/*.cu; do
  nvcc $FL $defs -c $f -o $out/$(basename $f .cu).o &
done
wait
nvcc $ARCH -shared -cudart static -o $out/libfxg.so $out/*.o paper_2603_12016_b200/build/fx_host.o paper_2603_12016_b200/build/engine.o paper_2603_12016_b200/build/fx_pack.o -lpthread -ldl -lrt
echo $out/libfxg.so
