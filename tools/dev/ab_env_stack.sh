#!/bin/bash
# A/B of an environment toggle on the layer-stack bench: bash tools/dev/ab_env_stack.sh CFG VAR
CFG=$1; VAR=$2
for r in 1 2; do for v in 0 1; do
  echo "$VAR=$v $CFG r$r: $(env $VAR=$v timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],3), {k: round(v,3) for k,v in d["per_category_ms"].items()})')"
done; done
