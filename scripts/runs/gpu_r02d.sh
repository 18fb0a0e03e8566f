#!/bin/bash
# Round-2 evidence call: GPU suite, tile-kernel variant A/B (cfg4), compute-sanitizer, and the
# full-length cfg2 parity job. Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_r02d.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputests_r02d.log 2>&1
echo "tests rc=$?"
STEPS=60 timeout 1500 bash scripts/exp_r02.sh > gpurun_out/exp_r02d.log 2>&1
echo "exp rc=$?"
timeout 2400 bash scripts/sanitize.sh > gpurun_out/sanitize_r02d.log 2>&1
echo "sanitize rc=$?"
timeout 1800 python scripts/cfg2_full_parity.py > gpurun_out/cfg2_full_r02d.json 2> gpurun_out/cfg2_full_r02d.err
echo "cfg2 full rc=$?"
