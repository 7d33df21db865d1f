#!/bin/bash
# ncu --set full with source of selected kernels of one P step (second rep).
# gpurun -- 'bash tools/dev/ncu_k.sh TAG REGEX SKIP COUNT [config]'
T=$1; R=$2; SK=${3:-3}; C=${4:-3}; CFG=${5:-paper}
O=gpurun_out/$T
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$R" -s $SK -c $C \
  -o $O/prof python tools/profile_step.py --config $CFG > $O/ncu.log 2>&1
tail -2 $O/ncu.log
ls -la $O
