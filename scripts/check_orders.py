"""Diagnostics: T after N steps under different element orders / tilings (deterministic mode),
each against the oracle replaying its own tiles, and against each other."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf, configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
case = configs.casting(n, jitter=0.2, seed=21, perm_seed=7, dt_safety=0.17)
res = {}
for no, eo in [("given", "given"), ("rcm", "min_node"), ("tile", "morton")]:
    opts = cf.SolveOptions(max_steps=steps, mode="deterministic", node_order=no, elem_order=eo)
    r = cf.solve(case.mesh, case.setup, opts)
    tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
    ref = orc.solve(case.mesh, case.setup, steps, blocks=tiles)
    res[eo] = r.T
    print(eo, "vs oracle same tiles: bitwise", np.array_equal(r.T, ref.T), "T range", r.T.min(), r.T.max(), flush=True)
for k in res:
    print(k, "vs given: max rel", float(np.max(np.abs(res[k] - res["given"]) / np.abs(res["given"]))),
          "nodes differing", int(np.sum(res[k] != res["given"])))
