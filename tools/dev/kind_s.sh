#!/bin/bash
# GEMM kinds on the step probe: bash tools/dev/kind_s.sh CFG S
CFG=$1; S=$2
for r in 1 2; do for K in tf32 f16x3 auto; do
  out=$(FFTCONV_B200_GEMM=$K timeout 200 python tools/dev/step_probe.py --config $CFG --S $S --reps 20 2>/dev/null)
  echo "$K $CFG S=$S r$r: $(echo "$out" | grep 'eager step flushed') | $(echo "$out" | grep -E '^  (forward|grad_input|grad_weight)' | awk '{print $3}' | tr '\n' ' ')"
done; done
