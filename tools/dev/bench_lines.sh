#!/bin/bash
# Bench lines only (no tests / ncu): bash tools/dev/bench_lines.sh TAG
O=gpurun_out/$1; mkdir -p $O
timeout 400 python bench.py > $O/bench_paper.json 2> $O/bench_paper.err
timeout 400 python bench.py --impl reference > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err
timeout 400 python bench.py --config wide > $O/bench_wide.json 2> $O/bench_wide.err
FFTCONV_B200_GEMM=tf32 timeout 400 python bench.py --config wide --no-cpu-baseline > $O/bench_wide_tf32.json 2> $O/bench_wide_tf32.err
timeout 600 python bench.py --config alex1 > $O/bench_alex1.json 2> $O/bench_alex1.err
timeout 400 python bench.py --config stack > $O/bench_stack.json 2> $O/bench_stack.err
timeout 400 python bench.py --config stack:alexnet-128 --steps 5 --warmup 3 > $O/bench_stack_alexnet.json 2> $O/bench_stack_alexnet.err
ls $O
