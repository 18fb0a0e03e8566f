import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
case = configs.casting(14, jitter=0.2, seed=3, perm_seed=9, dt_safety=0.14)
at = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=1, mode=sys.argv[1], elem_order="min_node", tile_elems=384))
print("ok", at.T[:3])
