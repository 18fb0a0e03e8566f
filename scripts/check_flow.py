"""Diagnostics: the bench/study Solver flow (step, time_phases, step, fields) on a multi-tile-per-CTA
mesh against the oracle replaying the same tiles."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf, configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
case = configs.casting(n, jitter=0.2, seed=21, perm_seed=7, dt_safety=0.17)
for persist in ["1", "0"]:
    os.environ["CF_TILE_PERSIST"] = persist
    opts = cf.SolveOptions(mode="deterministic")
    with cf.Solver(case.mesh, case.setup, opts) as sv:
        T0, _ = sv.fields(False)
        sv.step(5)
        T5, _ = sv.fields(False)
        ph = sv.time_phases(10)
        sv.step(20)
        T, _ = sv.fields(False)
        st = sv.stats()
    tiles, nt = cf.tile_map(case.mesh, case.setup, opts)
    ref5 = orc.solve(case.mesh, case.setup, 5, blocks=tiles).T
    ref = orc.solve(case.mesh, case.setup, 35, blocks=tiles).T
    print("persist", persist, "tiles", nt, "steps", st.step_index, "changed", int(np.sum(T != T0)), "/", T.size,
          "5-step bitwise", np.array_equal(T5, ref5), "35-step bitwise", np.array_equal(T, ref),
          "max rel", float(np.max(np.abs(T - ref) / np.abs(ref))), flush=True)
