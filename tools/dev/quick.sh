#!/bin/bash
# Quick GPU iteration: a parity subset, the step probe at P and W, and the
# P launch list.  gpurun --timeout 900 -- 'bash tools/dev/quick.sh TAG [pytest -k expr]'
T=${1:-q}
O=gpurun_out/$T
mkdir -p $O
K=${2:-}
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > $O/pytest.log 2>&1
else
  timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_workspace_reuse.py -m gpu -q -x > $O/pytest.log 2>&1
fi
tail -3 $O/pytest.log
timeout 300 python tools/dev/step_probe.py > $O/probe_paper.txt 2>&1
timeout 300 python tools/dev/step_probe.py --config wide --reps 10 > $O/probe_wide.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_paper.csv python tools/profile_step.py --reps 3 > /dev/null 2>&1
python tools/launch_sum.py $O/launches_paper.csv > $O/launch_sum.txt 2>&1
cat $O/probe_paper.txt $O/probe_wide.txt $O/launch_sum.txt
