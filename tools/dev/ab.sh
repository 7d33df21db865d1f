#!/bin/bash
# A/B of alternative library builds on the step probe: bash tools/dev/ab.sh TAG cfg lib1 lib2 ...
T=$1; CFG=$2; shift 2
O=gpurun_out/$T; mkdir -p $O
for round in 1 2; do
for L in "$@"; do
  n=$(basename $L .so)
  FFTCONV_B200_LIB=$L timeout 200 python tools/dev/step_probe.py --config $CFG --reps 30 > $O/${n}_${CFG}_$round.txt 2>&1
  echo "$n r$round: $(grep 'eager step flushed' $O/${n}_${CFG}_$round.txt) | $(grep -E '^  (forward|grad_input|grad_weight)' $O/${n}_${CFG}_$round.txt | awk '{print $2}' | tr '\n' ' ')"
done; done
