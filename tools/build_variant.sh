#!/bin/bash
# Build a variant of the CUDA library with extra compile definitions, for A/B
# runs (bench.py / tools with B200MOE_LIB=<path>):
#   tools/build_variant.sh <name> "-DFOO=1 -DBAR=2"  ->  paper_2412_09952_b200/lib/variants/<name>/libb200moe.so
set -e
cd "$(dirname "$0")/../paper_2412_09952_b200/csrc"
name=$1; defs=$2
out=../lib/variants/$name
mkdir -p $out/obj
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ftz=false -prec-div=true -prec-sqrt=true $defs"
for f in capi router permute router_bwd gemm upcycle model crc32c; do
  $NVCC $FLAGS -c $f.cu -o $out/obj/$f.o &
done
wait
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libb200moe.so $out/obj/*.o
rm -rf $out/obj
echo built $out/libb200moe.so
