#!/bin/bash
# sustained load (200 steps, the power cap engaged): 384-tet / 128-thread tiles vs 768-tet / 256-thread tiles
mkdir -p gpurun_out
for V in "384 128" "768 256" "384 128" "768 256"; do
  set -- $V
  CF_TILE_THREADS=$2 python bench.py --tile $1 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --compare-order none > gpurun_out/r02av.json 2> gpurun_out/r02av.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/r02av.json")); r=d["roofline"]
    print("tile $1 threads $2:", round(d["value"]/1e9,2), "G/s step", round(d["ms_per_step"],3), "ms", d["clocks"]["sm_mhz"], "MHz", d["clocks"]["power_w_max"], "W", d["clocks"]["reasons"])
except Exception as e:
    print("tile $1 threads $2 failed:", e)
PY
done
