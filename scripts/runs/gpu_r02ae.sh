#!/bin/bash
# atomic mode (fp64 RED on tile-shared nodes) beside deterministic mode, cfg5 and cfg2, same box
mkdir -p gpurun_out
for CFG in cfg5 cfg2; do for MODE in deterministic atomic; do
  python bench.py --config $CFG --mode $MODE --steps 40 --warmup 5 --no-cpu-baseline --compare-order none \
    > gpurun_out/r02ae_${CFG}_${MODE}.json 2> gpurun_out/r02ae_${CFG}_${MODE}.err
  python - <<PY
import json
d=json.load(open("gpurun_out/r02ae_${CFG}_${MODE}.json")); r=d["roofline"]
print("$CFG $MODE", round(d["value"]/1e9,2), "G/s step", round(d["ms_per_step"],4), "ms tile", r["kernel_ms"], "upd", r["update_ms"], "e2e", round(d["e2e"]["value"]/1e9,2), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "device GB", round(d["device_bytes"]/1e9,1))
PY
done; done
