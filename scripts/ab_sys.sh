#!/bin/bash
# A/B of systematic-codec library builds: put variants at build/ab/<name>.so (scripts/variant.sh), then run on the box.
mkdir -p gpurun_out/v8
timeout 600 python -m pytest tests/test_gpu_systematic.py -x -q > gpurun_out/v8/t.log 2>&1; echo "t rc=$?"; tail -1 gpurun_out/v8/t.log
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for v in new a0 m4 new a0 m4; do
  cp build/ab/$v.so paper_0907_1788_b200/libfntrs_b200.so
  timeout 300 python bench.py --codec systematic --steps 5 --no-cpu-baseline --e2e-stripes 0 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v',d['value'],d['encode_gbs'],d['decode_gbs'])"
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
