#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_multiprocess_gpu.py -q -x > gpurun_out/parity_r02k.log 2>&1
echo "parity rc=$?"; tail -2 gpurun_out/parity_r02k.log
for CFG in cfg5 cfg2; do
  for mode in gather copy; do
    if [ $mode = copy ]; then export CF_SLOT_COPY=1; else unset CF_SLOT_COPY; fi
    CFG=$CFG VARIANTS="base" VARIANTS5="none" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    \|none" | sed "s/^/$CFG $mode /"
  done
done
unset CF_SLOT_COPY
