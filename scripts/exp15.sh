#!/bin/bash
python bench.py > gpurun_out/bench_r01k.json 2> gpurun_out/bench_r01k.err; echo "cfg2 rc=$?"
python bench.py --config cfg4 --steps 100 --no-cpu-baseline > gpurun_out/bench_r01k_cfg4.json 2> gpurun_out/bench_r01k_cfg4.err; echo "cfg4 rc=$?"
python bench.py --config cfg5 --steps 40 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r01k_cfg5.json 2> gpurun_out/bench_r01k_cfg5.err; echo "cfg5 rc=$?"
