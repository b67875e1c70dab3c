#!/bin/bash
# A/B two library builds: ab_two.sh old.so new.so <rate_time shapes...>
old=$1; new=$2; shift 2
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for v in $old $new $old $new; do
  cp $v paper_0907_1788_b200/libfntrs_b200.so
  echo "== $v"; python scripts/rate_time.py "$@" 2>&1 | tail -n $#
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
