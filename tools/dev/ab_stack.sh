#!/bin/bash
# A/B of library builds on the layer-stack bench: bash tools/dev/ab_stack.sh CFG lib1 lib2 ...
CFG=$1; shift
for r in 1 2; do for L in "$@"; do
  echo "$(basename $L) $CFG r$r: $(FFTCONV_B200_LIB=$L timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],3), {k: round(v,3) for k,v in d["per_category_ms"].items()})')"
done; done
