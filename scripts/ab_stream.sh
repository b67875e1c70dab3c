#!/bin/bash
# A/B of streamed four-step library variants: ab_stream.sh lib1.so lib2.so ... (stream_ab.py per lib)
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for v in "$@"; do
  cp $v paper_0907_1788_b200/libfntrs_b200.so
  echo "== $v"; timeout 600 python scripts/stream_ab.py C4:64 C3:1 8,4 16,8 2>&1 | grep -E "stream|batched"
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
