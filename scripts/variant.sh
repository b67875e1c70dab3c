#!/bin/bash
# Build a library variant with extra nvcc flags for the decode / encode units:
#   variant.sh out.so "<codec_dec.cu flags>" "<codec_fast.cu flags>"
out=$1; fdec=$2; fenc=$3
set -e
NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC,-Wall -Iinclude -Ipaper_0907_1788_b200/csrc"
mkdir -p build/var
nvcc $NVFLAGS $fdec -c paper_0907_1788_b200/csrc/codec_dec.cu -o build/var/codec_dec.o &
nvcc $NVFLAGS $fenc -c paper_0907_1788_b200/csrc/codec_fast.cu -o build/var/codec_fast.o &
wait
objs=""
for o in build/*.o; do
  b=$(basename $o)
  if [ "$b" = codec_dec.o ] || [ "$b" = codec_fast.o ]; then objs="$objs build/var/$b"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs -Xcompiler -fPIC
echo built $out
