#!/bin/bash
for CFG in cfg5 cfg2; do
  for envs in "" "CF_BANK_PASSES=3" "CF_BANK_ITERS=8" "CF_BANK_PASSES=3 CF_BANK_ITERS=8"; do
    ( export $envs; CFG=$CFG VARIANTS="base" VARIANTS5="none" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    \|none" | sed "s/^/$CFG [$envs] /"; grep "device: rank plan" gpurun_out/exp_base.err | sed "s/^/   /" )
  done
done
