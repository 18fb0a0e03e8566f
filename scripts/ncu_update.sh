#!/bin/bash
TAG=${1:-x}
SMALL="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --phase-steps 2"
$SMALL > gpurun_out/plain_u_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:update_kernel -s 6 -c 1 -o gpurun_out/prof_update_${TAG} $SMALL > gpurun_out/ncu_u_${TAG}.log 2>&1
echo "ncu rc=$?"
