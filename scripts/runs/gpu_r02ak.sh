#!/bin/bash
# A/B: one warp polls the tile's mbarrier and the others wait in __syncthreads (CF_EXP_WAIT1) vs every thread polling
mkdir -p gpurun_out
CF_LIB_PATH=paper_1005_3158_b200/libcastfem_b200_wait1.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "casting or schedule" 2>&1 | tail -1
for CFG in cfg5 cfg2 cfg5; do
  CFG=$CFG VARIANTS="base wait1" VARIANTS5="none" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    \|none" | sed "s/^/$CFG /"
done
