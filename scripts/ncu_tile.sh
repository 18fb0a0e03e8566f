#!/bin/bash
# one ncu --set full capture of the tile kernel (cfg2, after the plain run exits 0)
TAG=${1:-x}
SMALL="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --phase-steps 2 $EXTRA"
$SMALL > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s ${SKIP:-7} -c 1 -o gpurun_out/prof_tile_${TAG} $SMALL > gpurun_out/ncu2_${TAG}.log 2>&1
echo "ncu rc=$?"
