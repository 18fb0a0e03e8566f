#!/bin/bash
for CFG in cfg5 cfg4 cfg2; do
  CFG=$CFG VARIANTS="base m5" VARIANTS5="none" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    \|none" | sed "s/^/$CFG /"
done
