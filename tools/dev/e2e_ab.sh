#!/bin/bash
# e2e A/B of library builds on one box: bash tools/dev/e2e_ab.sh lib1 lib2 ...
for r in 1 2 3; do for L in "$@"; do
  FFTCONV_B200_LIB=$L timeout 300 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', round(d['value'],4), 'e2e', round(d['e2e']['value'],3), 'h2d_alone', round(d['e2e']['pcie_floor_ms']['h2d_alone'],3))"
done; done
