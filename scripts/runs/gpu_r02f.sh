#!/bin/bash
mkdir -p gpurun_out
bash scripts/runs/gpu_r02e.sh > gpurun_out/r02f_devsetup.txt 2>&1
cat gpurun_out/r02f_devsetup.txt | grep -v "^\[cf setup\]" | tail -12
timeout 1500 python -m pytest tests -m gpu -q -x --durations=12 > gpurun_out/gputests_r02f.log 2>&1
echo "suite rc=$?"; tail -16 gpurun_out/gputests_r02f.log
VARIANTS="base" VARIANTS5="base m5" STEPS=60 timeout 1200 bash scripts/exp_r02.sh > gpurun_out/exp_r02f.log 2>&1
cat gpurun_out/exp_r02f.log | grep -v "^Traceback\|^  \|^json\|^    "
