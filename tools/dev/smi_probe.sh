#!/bin/bash
# Which nvidia-smi query stalls the host-driven stack iteration?  bash tools/dev/smi_probe.sh
FULL="clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu"
NOUTIL="clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,clocks.mem"
CLK="clocks.sm,clocks.max.sm"
for r in 1 2 3; do for name in FULL NOUTIL CLK; do
  q=${!name}
  echo "$name r$r: $(FFTCONV_BENCH_SMI_Q=$q timeout 300 python bench.py --config stack:alexnet-128 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"],3), round(d["per_category_ms"]["update_grad_input_ms"],3))')"
done; done
