#!/bin/bash
for CFG in ${CFGS:-cfg5 cfg2}; do
  for mode in off on; do
    if [ $mode = on ]; then export CF_L2_NEXT=1; else unset CF_L2_NEXT; fi
    CFG=$CFG VARIANTS="base" VARIANTS5="none" STEPS=${STEPS:-40} timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    \|none" | sed "s/^/$CFG l2next=$mode /"
  done
done
unset CF_L2_NEXT
