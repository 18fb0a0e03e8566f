import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
case = configs.casting(14, jitter=0.2, seed=3, perm_seed=9, dt_safety=0.14)
m = case.mesh
for order in ["min_node", "given", "morton"]:
    for no in ["tile", "given", "rcm"]:
        for te in [64, 128, 384, 1024]:
            at = cf.solve(m, case.setup, cf.SolveOptions(max_steps=1, mode="atomic", elem_order=order, node_order=no, tile_elems=te))
            de = cf.solve(m, case.setup, cf.SolveOptions(max_steps=1, mode="deterministic", elem_order=order, node_order=no, tile_elems=te))
            d = np.abs(at.T - de.T)
            print(order, no, te, "bad", int((d > 1e-9 * np.abs(de.T)).sum()), flush=True)
