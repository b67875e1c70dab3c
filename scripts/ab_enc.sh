for v in A B C D A; do
  cp build/vars/lib_$v.so paper_0907_1788_b200/libfntrs_b200.so
  echo "== $v"; python scripts/rate_time.py 128,256,2048,4096 128,256,2048,4096 2>&1 | tail -2
done
