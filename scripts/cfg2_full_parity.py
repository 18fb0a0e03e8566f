"""BASELINE configs[1] at its configured length: cfg2 (12.6 M tets, RCM-reordered) for the full
1000 steps on the B200, against the oracle replaying the same tiles (bitwise) and the reference
solver itself with one block (1e-9), the CPU runs concurrent. Too long for the -m gpu suite
(~10 min of CPU time); run once per round, result under profiles/:
    python scripts/cfg2_full_parity.py > profiles/r02_cfg2_full_parity.json"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402


def ref_steps(mesh, setup, steps):
    rb = orc.RefBench(mesh, setup)
    try:
        rb.steps(steps)
        return rb.T()
    finally:
        rb.close()


case = configs.config2()
steps = int(os.environ.get("STEPS", case.steps))
opts = cf.SolveOptions(max_steps=steps, node_order="rcm")
t0 = time.time()
with ThreadPoolExecutor(2) as ex:
    tiles, ntiles = cf.tile_map(case.mesh, case.setup, opts)
    f_or = ex.submit(orc.solve, case.mesh, case.setup, steps, tiles)
    f_ref = ex.submit(ref_steps, case.mesh, case.setup, steps)
    gpu = cf.solve(case.mesh, case.setup, opts)
    o = f_or.result()
    r = f_ref.result()
relr = float(np.max(np.abs(gpu.T - r) / np.abs(r)))
print(json.dumps({"workload": "cfg2", "node_order": "rcm", "steps": gpu.steps, "elements": case.mesh.element_count(),
                  "tiles": ntiles, "gpu_end_time": gpu.end_time, "oracle_end_time": o.time,
                  "bitwise_vs_oracle_same_tiles": bool(np.array_equal(gpu.T, o.T)),
                  "max_abs_diff_vs_oracle_same_tiles": float(np.abs(gpu.T - o.T).max()),
                  "max_rel_diff_vs_reference_1block": relr, "tolerance": 1e-9, "pass": relr <= 1e-9,
                  "T_min": float(gpu.T.min()), "T_max": float(gpu.T.max()),
                  "mushy_cast_nodes": int(np.sum((gpu.T > 821.0) & (gpu.T < 913.0))),
                  "wall_seconds": round(time.time() - t0, 1)}))
