#!/bin/bash
# Round evidence on one B200: GPU tests, bench lines, launch list, ncu --set full
# captures (summarised on the box by tools/ncu_summarize.py).
#   gpurun --timeout 3000 -- 'bash tools/evidence.sh r02_v1'
V=${1:-vX}
O=gpurun_out/ev_$V
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 400 python bench.py > $O/bench_paper.json 2> $O/bench_paper.err
timeout 400 python bench.py --impl reference > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err
timeout 400 python bench.py --config wide > $O/bench_wide.json 2> $O/bench_wide.err
FFTCONV_B200_GEMM=tf32 timeout 400 python bench.py --config wide --no-cpu-baseline > $O/bench_wide_tf32.json 2> $O/bench_wide_tf32.err
timeout 600 python bench.py --config alex1 > $O/bench_alex1.json 2> $O/bench_alex1.err
timeout 400 python bench.py --config stack > $O/bench_stack.json 2> $O/bench_stack.err
timeout 400 python bench.py --config stack:alexnet-128 --steps 5 --warmup 3 > $O/bench_stack_alexnet.json 2> $O/bench_stack_alexnet.err
for S in 16 32 64; do  # strong-scaling shards: per-rank step at S/N samples
  timeout 200 python tools/dev/step_probe.py --config wide --S $S --reps 20 > $O/probe_wide_S$S.txt 2>&1
  timeout 200 python tools/dev/step_probe.py --config paper --S $S --reps 20 > $O/probe_paper_S$S.txt 2>&1
done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_paper.csv \
  python tools/profile_step.py --reps 3 > /dev/null 2>&1
python tools/launch_sum.py $O/launches_paper.csv > $O/launch_sum_paper.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'r2c|cgemm|c2r' -s 9 -c 9 \
  -o $O/prof_paper python tools/profile_step.py --config paper > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'r2c|cgemm|c2r' -s 9 -c 9 \
  -o $O/prof_wide python tools/profile_step.py --config wide > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'128' -c 4 \
  -o $O/prof_alex1 python tools/profile_step.py --config alex1 --reps 1 --ops forward,grad_input > /dev/null 2>&1
for c in paper wide alex1; do
  python tools/ncu_summarize.py $c $O/prof_$c.ncu-rep $O/ncu_full_${c}_$V > /dev/null 2>&1
done
cp profiles/ncu_summary.json $O/ncu_summary.json
rm -f $O/prof_wide.ncu-rep $O/prof_alex1.ncu-rep
ls -la $O
