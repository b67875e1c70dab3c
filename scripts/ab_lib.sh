#!/bin/bash
# A/B two builds of the library on the same shapes: ab_lib.sh old.so new.so shapes...
old=$1; new=$2; shift 2
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for lib in $old $new; do
  cp $lib paper_0907_1788_b200/libfntrs_b200.so
  echo "== $lib"; python scripts/rate_time.py "$@" 2>&1
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
