#!/bin/bash
# refreshed studies with the final round-2 code: cfg3 ordering study, cfg2 1000-step parity, e2e at 200 steps
mkdir -p gpurun_out
timeout 1500 python scripts/reorder_study.py > gpurun_out/reorder_r02v.txt 2>&1; echo "reorder rc=$?"; tail -2 gpurun_out/reorder_r02v.txt | cut -c1-600
timeout 1800 python scripts/cfg2_full_parity.py > gpurun_out/cfg2_full_r02v.json 2> gpurun_out/cfg2_full_r02v.err; echo "cfg2 full rc=$?"; cat gpurun_out/cfg2_full_r02v.json
python bench.py --steps 200 --warmup 5 --no-cpu-baseline --compare-order none > gpurun_out/bench200_r02v.json 2> gpurun_out/bench200_r02v.err; echo "bench200 rc=$?"; cut -c1-300 gpurun_out/bench200_r02v.json
