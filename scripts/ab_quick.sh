#!/bin/bash
# A/B two library builds with quick_time.py: ab_quick.sh old.so new.so [CFG:S ...]
old=$1; new=$2; shift 2
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for lib in $old $new; do
  cp $lib paper_0907_1788_b200/libfntrs_b200.so
  echo "== $lib"; python scripts/quick_time.py "$@" 2>&1 | grep -v "^$"
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
