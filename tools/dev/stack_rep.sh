#!/bin/bash
# Repeated stack bench lines (outlier hunt): bash tools/dev/stack_rep.sh N [CFG]
N=${1:-3}; CFG=${2:-stack:alexnet-128}
for i in $(seq $N); do
  timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3), {k: round(v,3) for k,v in d["per_category_ms"].items()}, d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"), round(d["wall_ms_incl_param_upload"],1))'
done
