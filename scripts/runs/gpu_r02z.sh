#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "schedule or casting" 2>&1 | tail -2
for CFG in cfg5 cfg2 cfg5; do
  CFG=$CFG VARIANTS="prev base" VARIANTS5="none" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    \|none" | sed "s/^/$CFG /"
done
