"""Diagnostics: BASELINE configs[2] (cfg3) under the three orderings, each against the oracle
replaying its own tiles (bitwise), after N steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf, configs
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
case = configs.config3()
res = {}
for no, eo in [("given", "given"), ("rcm", "min_node"), ("tile", "morton")]:
    opts = cf.SolveOptions(max_steps=steps, mode="deterministic", node_order=no, elem_order=eo)
    r = cf.solve(case.mesh, case.setup, opts)
    tiles, nt = cf.tile_map(case.mesh, case.setup, opts)
    ref = orc.solve(case.mesh, case.setup, steps, blocks=tiles)
    res[eo] = r.T
    print(eo, nt, "tiles; vs oracle same tiles: bitwise", np.array_equal(r.T, ref.T), "nodes differing",
          int(np.sum(r.T != ref.T)), "max rel", float(np.max(np.abs(r.T - ref.T) / np.abs(ref.T))), flush=True)
for k in res:
    print(k, "vs given: nodes differing", int(np.sum(res[k] != res["given"])))
