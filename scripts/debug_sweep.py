import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
from oracle import oracle as orc
for n in [int(x) for x in sys.argv[1].split(",")]:
    case = configs.casting(n, dt_safety=0.14)
    for mode in ["atomic", "deterministic"]:
        for tile in [256, 1024]:
            try:
                r = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=3, mode=mode, tile_elems=tile))
                msg = "ok"
                if n <= 40:
                    o = orc.solve(case.mesh, case.setup, 3)
                    msg += f" rel={np.max(np.abs(r.T-o.T)/np.abs(o.T)):.2e}"
            except Exception as e:
                msg = f"FAIL {e}"
            print(n, mode, tile, msg, flush=True)
