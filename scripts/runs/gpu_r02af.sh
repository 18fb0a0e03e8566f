#!/bin/bash
# atomic mode with interleaved (c, r) accumulators: atomic-mode tests, then the r02ae comparison again
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_multiprocess_gpu.py tests/test_gpu_fuzz.py -q -x -m gpu 2>&1 | tail -3
for CFG in cfg5 cfg2; do for MODE in atomic; do
  python bench.py --config $CFG --mode $MODE --steps 40 --warmup 5 --no-cpu-baseline --compare-order none \
    > gpurun_out/r02af_${CFG}_${MODE}.json 2> gpurun_out/r02af_${CFG}_${MODE}.err
  python - <<PY
import json
d=json.load(open("gpurun_out/r02af_${CFG}_${MODE}.json")); r=d["roofline"]
print("$CFG $MODE", round(d["value"]/1e9,2), "G/s step", round(d["ms_per_step"],4), "ms tile", r["kernel_ms"], "upd", r["update_ms"], "e2e", round(d["e2e"]["value"]/1e9,2), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "device GB", round(d["device_bytes"]/1e9,1))
PY
done; done
