#!/bin/bash
# A/B several library builds on the same shapes: ab_multi.sh "a.so b.so ..." shapes...
libs=$1; shift
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for lib in $libs; do
  cp $lib paper_0907_1788_b200/libfntrs_b200.so
  echo "== $lib"; python scripts/rate_time.py "$@" 2>&1 | grep -v Warn
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
