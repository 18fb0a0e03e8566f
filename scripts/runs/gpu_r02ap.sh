#!/bin/bash
# tile-size sweep at cfg5 on the final code (the autotuner's candidates and neighbours)
mkdir -p gpurun_out
for T in 192 320 384 448 768; do
  python bench.py --tile $T --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --compare-order none > gpurun_out/r02ap_tile$T.json 2> gpurun_out/r02ap_tile$T.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/r02ap_tile$T.json")); r=d["roofline"]
    print("tile_elems $T:", round(d["value"]/1e9,2), "G/s step", round(d["ms_per_step"],3), "ms tile", r["kernel_ms"], "upd", r["update_ms"], "tiles", d["tiles"], "slots", d["total_slots"], d["clocks"]["sm_mhz"])
except Exception as e:
    print("tile_elems $T failed:", e)
PY
done
