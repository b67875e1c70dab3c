#!/bin/bash
# e2e pipeline chunk / stream sweep (the line's e2e only)
for opt in "--e2e-chunk 256 --e2e-streams 4" "--e2e-chunk 128 --e2e-streams 4" "--e2e-chunk 128 --e2e-streams 8" "--e2e-chunk 256 --e2e-streams 8" "--e2e-chunk 512 --e2e-streams 4" "--e2e-chunk 64 --e2e-streams 8" "--e2e-chunk 256 --e2e-streams 4"; do
  python bench.py --steps 5 --warmup 3 --stripes 1024 --no-cpu-baseline --sweep none $opt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read())['e2e']; print('$opt', d['value'], d['pcie_h2d_gbs'], d['pcie_d2h_gbs'], d['pcie_peak_d2h_gbs'])"
done
