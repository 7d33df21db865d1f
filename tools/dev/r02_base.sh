O=gpurun_out/r02_base
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 400 python bench.py > $O/bench_paper.json 2> $O/bench_paper.err
timeout 400 python bench.py --config wide > $O/bench_wide.json 2> $O/bench_wide.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_paper.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
cat $O/bench_paper.json
