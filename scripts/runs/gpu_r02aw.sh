#!/bin/bash
# FMA contraction (-fmad=true build) vs the bitwise build (-fmad=false), sustained load (200 steps) and 20 steps;
# deviation of the FMA build from the oracle on a small casting
mkdir -p gpurun_out
CF_LIB_PATH=paper_1005_3158_b200/libcastfem_b200_fma.so python - <<'PY'
import numpy as np
from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf, configs
case = configs.casting(24, jitter=0.1, seed=3, dt_safety=0.14)
opts = cf.SolveOptions(max_steps=300, tile_elems=384)
g = cf.solve(case.mesh, case.setup, opts)
tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
r = orc.solve(case.mesh, case.setup, 300, blocks=tiles)
print("fma build vs oracle, casting24 300 steps: max rel", float(np.max(np.abs(g.T - r.T) / np.abs(r.T))), "bitwise", bool(np.array_equal(g.T, r.T)))
g2 = cf.solve(case.mesh, case.setup, opts)
print("fma build run-to-run bitwise:", bool(np.array_equal(g.T, g2.T)))
PY
for S in 200 20; do for v in base fma base fma; do
  lib=libcastfem_b200_$v.so; [ $v = base ] && lib=libcastfem_b200.so
  CF_LIB_PATH=paper_1005_3158_b200/$lib python bench.py --steps $S --warmup 5 --no-cpu-baseline --no-e2e --compare-order none > gpurun_out/r02aw.json 2> gpurun_out/r02aw.err
  python - <<PY
import json
try:
    d=json.load(open("gpurun_out/r02aw.json")); r=d["roofline"]
    print("$v steps $S:", round(d["value"]/1e9,2), "G/s step", round(d["ms_per_step"],3), "ms tile", r["kernel_ms"], d["clocks"]["sm_mhz"], "MHz", d["clocks"]["power_w_max"], "W")
except Exception as e:
    print("$v steps $S failed:", e)
PY
done; done
