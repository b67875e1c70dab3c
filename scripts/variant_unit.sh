#!/bin/bash
# Build a library variant with extra nvcc flags for one unit:
#   variant_unit.sh out.so <unit (e.g. codec_large)> "<flags>"
out=$1; unit=$2; flags=$3
set -e
NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC,-Wall -Iinclude -Ipaper_0907_1788_b200/csrc"
mkdir -p build/var
nvcc $NVFLAGS $flags -c paper_0907_1788_b200/csrc/$unit.cu -o build/var/$unit.o
objs=""
for o in build/*.o; do
  b=$(basename $o)
  if [ "$b" = $unit.o ]; then objs="$objs build/var/$b"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs -Xcompiler -fPIC
echo built $out
