"""Strong-scaling proxy at the gate configuration on ONE GPU: cfg5 (805 M tets, device-generated
mesh) split by RCB into R parts, all R ranks in one process over the in-process transport (device
copies; no cross-rank waits). The R ranks' kernels run one after another on the one GPU, so
T(R=1) / T(R) estimates the parallel efficiency of R GPUs before any interconnect cost (the
per-step exchange at R = 8 is ~3 MB per GPU). python scripts/inprocess_decomposition_fixture.py cfg5 "1 8" 20"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
Rs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1 8").split()]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
dc = configs.device_case(cfg)
out = {"config": cfg, "steps": steps, "transport": "in-process (one GPU)"}
ref = None
for R in Rs:
    t0 = time.time()
    with cf.Solver(None, dc.setup, cf.SolveOptions(world_size=R, local_ranks=R, rank=0), fixture=dc.spec) as sv:
        setup = time.time() - t0
        E = sv.stats().n_elems_global
        sv.step(3)
        before = sv.stats().loop_seconds
        sv.step(steps)
        secs = sv.stats().loop_seconds - before
        T = sv.fields(False)[0]
        ph = sv.time_phases(5)
        st = sv.stats()
    if ref is None:
        ref = T
    out[f"R={R}"] = {"element_updates_per_s": E * steps / secs, "ms_per_step": 1e3 * secs / steps,
                     "setup_s": round(setup, 2), "device_bytes": st.device_bytes,
                     "phases_ms (tile, pack, exchange, update)": [round(float(x), 4) for x in ph],
                     "max_rel_vs_first": float(np.max(np.abs(T - ref) / np.abs(ref)))}
    print(R, out[f"R={R}"], flush=True)
r1 = out.get("R=1")
for R in Rs:
    if r1 and R > 1:
        out[f"R={R}"]["efficiency_proxy"] = r1["ms_per_step"] / out[f"R={R}"]["ms_per_step"]
print(json.dumps(out))
