#!/bin/bash
# device setup pipeline: its GPU tests first, then a cfg2 / cfg5 creation check
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_devsetup.py -q -x --durations=5 > gpurun_out/devsetup_tests.log 2>&1
echo "devsetup tests rc=$?"
tail -30 gpurun_out/devsetup_tests.log
CF_TRACE_SETUP=1 timeout 600 python scripts/devsetup_cfg.py cfg2 > gpurun_out/devsetup_cfg2.json 2> gpurun_out/devsetup_cfg2.err
echo "cfg2 rc=$?"; cat gpurun_out/devsetup_cfg2.json; tail -30 gpurun_out/devsetup_cfg2.err
CF_TRACE_SETUP=1 timeout 900 python scripts/devsetup_cfg.py cfg5 > gpurun_out/devsetup_cfg5.json 2> gpurun_out/devsetup_cfg5.err
echo "cfg5 rc=$?"; cat gpurun_out/devsetup_cfg5.json; tail -30 gpurun_out/devsetup_cfg5.err
