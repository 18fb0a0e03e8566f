"""Diagnostics: the decomposed (multi-rank) data path on ONE GPU, all ranks in one process over
the in-process transport (device copies; no cross-rank waits): cfg4 (256^3 casting, 100.7 M tets)
split by RCB into R parts, R = 1, 2, 8. Whole-mesh element-updates/s per R shows the cost of the
decomposition itself (per-rank launches, border/interior split, pack + exchange copies, shared
nodes merged across ranks); results are bitwise identical across R only up to summation order,
so T is compared within 1e-9 relative."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
case = configs.casting(n, dt_safety=configs.DT_SAFETY["cfg4"], steps=steps)
E = case.mesh.element_count()
out = {"mesh": f"casting {n}^3", "elements": E, "steps": steps}
ref = None
for R in [int(x) for x in os.environ.get("RANKS", "1 2 8").split()]:
    t0 = time.time()
    opts = cf.SolveOptions(world_size=R, local_ranks=R, rank=0)
    with cf.Solver(case.mesh, case.setup, opts) as sv:
        setup = time.time() - t0
        sv.step(3)
        before = sv.stats().loop_seconds
        sv.step(steps)
        secs = sv.stats().loop_seconds - before
        T, _ = sv.fields(False)
        ph = sv.time_phases(10)
    if ref is None:
        ref = T
    out[f"R={R}"] = {"element_updates_per_s": E * steps / secs, "ms_per_step": 1e3 * secs / steps,
                     "setup_s": setup,
                     "phases_ms (tile, pack, exchange, update)": [float(x) for x in ph], "max_rel_vs_R1": float(np.max(np.abs(T - ref) / np.abs(ref)))}
    print(R, out[f"R={R}"], flush=True)
print(json.dumps(out))
