#!/bin/bash
# A/B: streaming cache hints (CF_EXP_HINTS: st.cs on partials / Tn / slot copies, ld.cs on the update's partial reads)
mkdir -p gpurun_out
for CFG in cfg5 cfg2 cfg5; do
  CFG=$CFG VARIANTS="base hints" VARIANTS5="none" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    \|none" | sed "s/^/$CFG /"
done
