#!/bin/bash
# A/B several library builds on the same shapes (rate_time.py), two rounds:
#   ab_n.sh "shape1 shape2" lib1.so lib2.so ...
shapes=$1; shift
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for round in 1 2; do
  for v in "$@"; do
    cp $v paper_0907_1788_b200/libfntrs_b200.so
    echo "== $v"; python scripts/rate_time.py $shapes 2>&1 | grep GB/s
  done
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
