#!/bin/bash
# A/B of library builds on the step probe for one config and batch:
#   bash tools/dev/ab_s.sh CFG S lib1 lib2 ...   (S = 0: the config's own batch)
CFG=$1; S=$2; shift 2
for r in 1 2; do for L in "$@"; do
  out=$(FFTCONV_B200_LIB=$L timeout 200 python tools/dev/step_probe.py --config $CFG --S $S --reps 20 2>/dev/null)
  echo "$(basename $L) $CFG S=$S r$r: $(echo "$out" | grep 'eager step flushed') | $(echo "$out" | grep -E '^  (forward|grad_input|grad_weight)' | awk '{print $3}' | tr '\n' ' ')"
done; done
