#!/bin/bash
# Library variant with extra nvcc flags for ONE translation unit (others from build/):
#   variant_tu.sh out.so <unit, e.g. codec_large> "<flags>"
out=$1; unit=$2; flags=$3
set -e
NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC,-Wall -Iinclude -Ipaper_0907_1788_b200/csrc"
d=build/var_$(basename $out .so); mkdir -p $d
nvcc $NVFLAGS $flags -c paper_0907_1788_b200/csrc/$unit.cu -o $d/$unit.o
objs=""
for o in build/*.o; do
  b=$(basename $o)
  if [ "$b" = $unit.o ]; then objs="$objs $d/$b"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs -Xcompiler -fPIC
echo built $out
