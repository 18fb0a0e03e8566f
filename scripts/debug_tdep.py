import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf
from oracle import oracle as orc
m = cf.generate_fixture("cube", 8)
x0 = np.all(m.nodes[m.facets][:, :, 0] == 0.0, axis=1)
m.facet_tag = np.where(x0, 1, 0).astype(np.int32); m.tags = ["outer", "hot"]
for label, ctab, ktab, L, dirichlet in [
        ("const+dir", 450.0, 45.0, 2.0e5, True), ("tdep c only", [(300.0, 450.0), (900.0, 700.0)], 45.0, 2.0e5, False),
        ("tdep k only", 450.0, [(300.0, 45.0), (900.0, 30.0)], 2.0e5, False), ("tdep both nolatent", [(300.0, 450.0), (900.0, 700.0)], [(300.0, 45.0), (900.0, 30.0)], 0.0, False),
        ("tdep both", [(300.0, 450.0), (900.0, 700.0)], [(300.0, 45.0), (900.0, 30.0)], 2.0e5, False)]:
    mat = cf.MaterialTable.make(rho=7800.0, c=ctab, k=ktab, latent_heat=L, solidus=700.0, liquidus=760.0, T0=650.0)
    bcs = {"outer": cf.BoundaryCondition("flux", h=50.0, t_inf=300.0)}
    bcs["hot"] = cf.BoundaryCondition("fixed", fixed_T=cf.PiecewiseLinear([0.0, 50.0], [650.0, 950.0])) if dirichlet else cf.BoundaryCondition("flux", h=5000.0, t_inf=950.0)
    setup = cf.SimulationSetup(materials=[mat], boundary_conditions=bcs, solver=cf.SolverConfig(dt_safety=0.1))
    for steps in [2, 10]:
        for tile in [128, 4096 // 4]:
            gpu = cf.solve(m, setup, cf.SolveOptions(max_steps=steps, tile_elems=tile))
            ref = orc.solve(m, setup, steps)
            d = np.abs(gpu.T - ref.T)
            bad = np.where(d > 0)[0]
            print(label, steps, tile, "nbad", len(bad), "max", d.max(), "dt", gpu.end_time == ref.time, bad[:6])
