import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
from oracle import oracle as orc
def rel(a, b): return float(np.max(np.abs(a - b) / np.abs(b)))
case = configs.casting(12, jitter=0.15, seed=2, dt_safety=0.14)
for ranks in [2]:
    parts = cf.partition_rcb(case.mesh, ranks)
    for steps in [1, 2, 5, 30]:
        opts = cf.SolveOptions(max_steps=steps, mode="deterministic", tile_elems=256, world_size=ranks, local_ranks=ranks)
        gpu = cf.solve(case.mesh, case.setup, opts)
        tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
        ref = orc.solve(case.mesh, case.setup, steps, blocks=tiles, parts=parts)
        single = orc.solve(case.mesh, case.setup, steps)
        d = np.abs(gpu.T - ref.T)
        print(ranks, steps, "vs parts-oracle", rel(gpu.T, ref.T), "nbad", int((d > 0).sum()), "vs single", rel(gpu.T, single.T), "oracle parts vs single", rel(ref.T, single.T))
# dirichlet/tdep
m = cf.generate_fixture("cube", 8)
x0 = np.all(m.nodes[m.facets][:, :, 0] == 0.0, axis=1)
m.facet_tag = np.where(x0, 1, 0).astype(np.int32); m.tags = ["outer", "hot"]
mat = cf.MaterialTable.make(rho=7800.0, c=[(300.0, 450.0), (900.0, 700.0)], k=[(300.0, 45.0), (900.0, 30.0)], latent_heat=2.0e5, solidus=700.0, liquidus=760.0, T0=650.0)
setup = cf.SimulationSetup(materials=[mat], boundary_conditions={"outer": cf.BoundaryCondition("flux", h=50.0, t_inf=300.0), "hot": cf.BoundaryCondition("fixed", fixed_T=cf.PiecewiseLinear([0.0, 50.0], [650.0, 950.0]))}, solver=cf.SolverConfig(dt_safety=0.1))
for steps in [1, 2, 3, 10, 60]:
    gpu = cf.solve(m, setup, cf.SolveOptions(max_steps=steps, tile_elems=128))
    ref = orc.solve(m, setup, steps)
    d = np.abs(gpu.T - ref.T)
    print("tdep", steps, rel(gpu.T, ref.T), int((d > 0).sum()), gpu.end_time - ref.time, "dt", ref.dt)
