#!/bin/bash
# One gpurun call (round 2): the driver-shaped bench line at cfg5, the reference arm, the ncu
# launch list of the step kernels and one ncu --set full capture of the tile kernel (each ncu
# pass only after its command exited 0 without ncu). TAG names the outputs.
TAG=${1:-r02}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/reference_${TAG}.json 2> gpurun_out/reference_${TAG}.err
echo "reference rc=$?"
SMALL="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --phase-steps 1 --compare-order none"
K='regex:tile_kernel|update_kernel|advance_kernel'
$SMALL > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 30 --csv --log-file gpurun_out/launches_${TAG}.csv $SMALL > gpurun_out/ncu1_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s ${SKIP:-4} -c 1 -o gpurun_out/prof_tile_${TAG} $SMALL > gpurun_out/ncu2_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:update_kernel -s ${SKIP:-4} -c 1 -o gpurun_out/prof_update_${TAG} $SMALL > gpurun_out/ncu3_${TAG}.log 2>&1
echo "ncu rc=$?"
