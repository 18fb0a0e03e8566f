#!/bin/bash
# One gpurun call: bench line (+ reference arm), ncu launch list, ncu --set full of the top kernel.
set -x
TAG=${1:-r01}
SMALL="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --phase-steps 2"
python bench.py --steps ${STEPS:-200} --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reference_${TAG}.json 2> gpurun_out/reference_${TAG}.err
echo "reference rc=$?"
$SMALL > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_${TAG}.csv $SMALL > gpurun_out/ncu1_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s ${SKIP:-7} -c 1 -o gpurun_out/prof_tile_${TAG} $SMALL > gpurun_out/ncu2_${TAG}.log 2>&1
echo "ncu rc=$?"
