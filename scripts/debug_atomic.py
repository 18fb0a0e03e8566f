import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
from oracle import oracle as orc
case = configs.casting(14, jitter=0.2, seed=3, perm_seed=9, dt_safety=0.14)
m = case.mesh
for steps in [1, 2, 5]:
    for order in ["morton", "min_node"]:
        o = cf.SolveOptions(max_steps=steps, mode="atomic", elem_order=order)
        at = cf.solve(m, case.setup, o)
        de = cf.solve(m, case.setup, cf.SolveOptions(max_steps=steps, mode="deterministic", elem_order=order))
        tiles, nt = cf.tile_map(m, case.setup, o)
        ntiles = np.zeros(m.node_count(), int)
        for n in range(m.node_count()):
            pass
        # node -> set of tiles
        tt = np.repeat(tiles, 4); nn = m.tets.reshape(-1)
        pairs = np.unique(nn * 100000 + tt)
        cnt = np.bincount(pairs // 100000, minlength=m.node_count())
        d = np.abs(at.T - de.T)
        bad = np.where(d > 1e-9 * np.abs(de.T))[0]
        print(steps, order, "tiles", nt, "bad", len(bad), "max", d.max(), "tilecount of bad:", np.bincount(cnt[bad]) if len(bad) else "-", "all:", np.bincount(cnt))
