#!/bin/bash
# A/B of library builds on the step probe for one config: bash tools/dev/ab_cfg.sh CFG lib1 lib2 ...
CFG=$1; shift
for r in 1 2; do for L in "$@"; do
  echo "$(basename $L) $CFG r$r: $(FFTCONV_B200_LIB=$L timeout 200 python tools/dev/step_probe.py --config $CFG --reps 20 2>/dev/null | grep 'eager step flushed')"
done; done
