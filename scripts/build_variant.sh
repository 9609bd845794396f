#!/bin/bash
# usage: build_variant.sh <suffix> <extra nvcc flags...>  -> paper_2211_12265_b200/libdilithium_b200_<suffix>.so
set -e
sfx=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_2211_12265_b200/csrc
tmp=$(mktemp -d)
for f in engine keygen verify sign peaks; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $src/$f.cu -o $tmp/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $root/paper_2211_12265_b200/libdilithium_b200_$sfx.so $tmp/*.o
rm -rf $tmp
echo built libdilithium_b200_$sfx.so
