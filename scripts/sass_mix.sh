#!/bin/bash
# Static SASS opcode mix of one kernel: sass_mix.sh <source.cu> <kernel-name regex> [extra nvcc flags]
# (compiles the source alone to a cubin; counts are static, not executed)
src=$1; pat=$2; shift 2
out=/tmp/sass_mix.cubin
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -cubin \
     -Ipaper_0907_1788_b200/csrc "$@" -o $out $src || exit 1
fn=$(cuobjdump -symbols $out | grep -o "_Z[^ ]*" | grep -E "$pat" | grep -v '\$' | head -1)
echo "$fn"
cuobjdump -sass -fun "$fn" $out > /tmp/sass_mix.txt
grep -oE "^\s+/\*[0-9a-f]+\*/\s+[@!A-Z0-9P_ ]*[A-Z][A-Z0-9_.]+" /tmp/sass_mix.txt | awk '{ op=$2; if (op ~ /^@/) op=$3; print op }' \
  | sort | uniq -c | sort -rn | head -${TOP:-25}
echo "total $(grep -cE '^\s+/\*[0-9a-f]+\*/' /tmp/sass_mix.txt)"
