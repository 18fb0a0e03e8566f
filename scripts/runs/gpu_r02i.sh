#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_devsetup.py -q -x > gpurun_out/devsetup_r02i.log 2>&1
echo "devsetup rc=$?"; tail -3 gpurun_out/devsetup_r02i.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02i.json 2> gpurun_out/bench_r02i.err
echo "bench rc=$?"; cat gpurun_out/bench_r02i.json; tail -3 gpurun_out/bench_r02i.err
python bench.py --impl reference --steps 20 --warmup 5 --ref-blocked > gpurun_out/reference_r02i.json 2> gpurun_out/reference_r02i.err
echo "reference rc=$?"; cat gpurun_out/reference_r02i.json; tail -3 gpurun_out/reference_r02i.err
