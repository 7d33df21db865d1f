#!/bin/bash
# Stack and P bench lines with the two-rate clock sampler (outlier check).
for r in 1 2 3 4; do
  echo "stack r$r: $(timeout 300 python bench.py --config stack:alexnet-128 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],3), round(d["per_category_ms"]["update_grad_input_ms"],3), d["clocks"])')"
done
for r in 1 2; do
  echo "P r$r: $(timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],4), d["clocks"])')"
done
