import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf
from oracle import oracle as orc
m = cf.generate_fixture("cube", 8)
x0 = np.all(m.nodes[m.facets][:, :, 0] == 0.0, axis=1)
m.facet_tag = np.where(x0, 1, 0).astype(np.int32); m.tags = ["outer", "hot"]
mat = cf.MaterialTable.make(rho=7800.0, c=450.0, k=[(300.0, 45.0), (900.0, 30.0)], latent_heat=2.0e5, solidus=700.0, liquidus=760.0, T0=650.0)
bcs = {"outer": cf.BoundaryCondition("flux", h=50.0, t_inf=300.0), "hot": cf.BoundaryCondition("flux", h=5000.0, t_inf=950.0)}
setup = cf.SimulationSetup(materials=[mat], boundary_conditions=bcs, solver=cf.SolverConfig(dt_safety=0.1))
for tile in [128, 1024]:
    o = cf.SolveOptions(max_steps=10, tile_elems=tile)
    tiles, _ = cf.tile_map(m, setup, o)
    for name, f in (("gpu", lambda: cf.solve(m, setup, o).T), ("oracle-tiles", lambda: orc.solve(m, setup, 10, blocks=tiles).T)):
        try: T = f(); print(tile, name, "ok", T[:2])
        except Exception as e: print(tile, name, "raised:", e)
