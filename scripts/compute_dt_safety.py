"""Measures lambda_max of M_L^-1 (K + H) by power iteration on the GPU for the
BASELINE configs and prints dt_safety = 0.9 * 2 / lambda_max / min_e(rho c l^2/k)
(SURVEY §0 trap 2). The printed values are recorded in
paper_1005_3158_b200/configs.py:DT_SAFETY with this script as provenance."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402

ITERS = int(os.environ.get("LAMBDA_ITERS", "3000"))
out = {}
names = sys.argv[1:] or ["cfg1", "cfg3", "cfg2", "cfg4", "cfg5"]
for name, make in [(k, configs.CONFIGS[k]) for k in names]:
    t0 = time.time()
    case = make()
    with cf.Solver(case.mesh, case.setup, cf.SolveOptions(max_steps=0)) as s:
        lam, e13 = s.estimate_lambda_max(ITERS)
    ds = configs.dt_safety_from_lambda(lam, e13)
    out[name] = {"lambda_max": lam, "eq13_min": e13, "ratio_true_over_eq13": 2.0 / lam / e13, "dt_safety": ds,
                 "dt": ds * e13, "iterations": ITERS, "seconds": round(time.time() - t0, 1)}
    print(name, json.dumps(out[name]), flush=True)
print(json.dumps(out))
