#!/bin/bash
# A/B library builds with quick_time.py: ab_quick.sh "a.so b.so ..." [CFG:S ...]
libs=$1; shift
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for lib in $libs; do
  cp $lib paper_0907_1788_b200/libfntrs_b200.so
  echo "== $lib"; python scripts/quick_time.py "$@" 2>&1 | grep -v "^$"
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
