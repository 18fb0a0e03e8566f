#!/bin/bash
# 768-tet tiles with 256-thread CTAs (2 CTAs x 8 warps per SM) re-measured on the final code, cfg5 and cfg2
mkdir -p gpurun_out
for CFG in cfg5 cfg2; do for V in "384 128" "768 256" "768 128" "384 128"; do
  set -- $V
  CF_TILE_THREADS=$2 python bench.py --config $CFG --tile $1 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --compare-order none > gpurun_out/r02aq.json 2> gpurun_out/r02aq.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/r02aq.json")); r=d["roofline"]
    print("$CFG tile $1 threads $2:", round(d["value"]/1e9,2), "G/s step", round(d["ms_per_step"],4), "ms tile", r["kernel_ms"], "upd", r["update_ms"], d["clocks"]["sm_mhz"])
except Exception as e:
    print("$CFG tile $1 threads $2 failed:", e)
PY
done; done
