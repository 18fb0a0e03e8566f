#!/bin/bash
# Closing evidence on the final round-2 tree (TAG r02ac): GPU suite + smoke, driver-shaped bench and
# reference arm at cfg5, ncu launch list + --set full captures of both step kernels, cfg2 bench
# (RCM-reordered mesh), cfg2 1000-step parity, cfg5 at its configured 200 steps.
export TAG=r02ac
bash scripts/runs/gpu_r02n.sh > gpurun_out/r02ac_main.log 2>&1; tail -c 1500 gpurun_out/r02ac_main.log
python bench.py --config cfg2 --steps 1000 --warmup 5 > gpurun_out/bench_cfg2_r02ac.json 2> gpurun_out/bench_cfg2_r02ac.err; echo "cfg2 bench rc=$?"
python bench.py --steps 200 --warmup 5 --no-cpu-baseline --compare-order none > gpurun_out/bench200_r02ac.json 2> gpurun_out/bench200_r02ac.err; echo "bench200 rc=$?"
timeout 1800 python scripts/cfg2_full_parity.py > gpurun_out/cfg2_full_r02ac.json 2> gpurun_out/cfg2_full_r02ac.err; echo "cfg2 full rc=$?"; cat gpurun_out/cfg2_full_r02ac.json
