#!/bin/bash
# driver-shaped bench (cfg5, device-generated mesh) + 5-CTA variant A/B on cfg2 and cfg5
mkdir -p gpurun_out
/usr/bin/time -v python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err
echo "bench rc=$?"; cat gpurun_out/bench_r02g.json; grep -E "Elapsed|Maximum resident" gpurun_out/bench_r02g.err
CFG=cfg2 VARIANTS="base m5" VARIANTS5="m5" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    " | sed "s/^/cfg2 /"
CFG=cfg5 VARIANTS="base m5" VARIANTS5="m5" STEPS=40 timeout 1200 bash scripts/exp_r02.sh 2>&1 | grep -v "^Traceback\|^  \|^json\|^    " | sed "s/^/cfg5 /"
