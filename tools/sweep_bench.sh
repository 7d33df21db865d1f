#!/bin/bash
# Bench lines for every BASELINE single-GPU configuration: configs[0] (small),
# configs[1] (paper), all 18 configs[2] points, configs[3] on one GPU (wide,
# auto and 3xTF32), configs[4]'s first layer (alex1) and the stacks.
#   gpurun --timeout 3000 -- 'bash tools/sweep_bench.sh TAG'
T=${1:-sweep}
O=gpurun_out/$T
mkdir -p $O
run() {  # name, args...
  local name=$1; shift
  timeout 600 python bench.py "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$? $(head -c 160 $O/$name.json)"
}
run small --config small
run paper --config paper
for n in 16 32 64; do for k in 3 5 7 9 11 13; do
  run sweep_${n}_${k} --config sweep:$n,$k --steps 10
done; done
run wide --config wide --steps 10
FFTCONV_B200_GEMM=tf32 run wide_tf32 --config wide --steps 10
run alex1 --config alex1 --steps 10
run reference_small --config small --impl reference --steps 3
run reference_paper --config paper --impl reference --steps 3
