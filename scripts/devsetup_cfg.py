"""Device setup pipeline on a BASELINE config: plan creation time and host peak RSS with the
mesh generated on the device (no host mesh), a few steps, and (cfg2/cfg4) bitwise equality with
the plan built from the host fixture.  python scripts/devsetup_cfg.py cfg5"""
import json
import os
import resource
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
order = sys.argv[2] if len(sys.argv) > 2 else "rcm"
dc = configs.device_case(name)
rss0 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
t0 = time.time()
s = cf.Solver(None, dc.setup, cf.SolveOptions(node_order=order), fixture=dc.spec)
t_setup = time.time() - t0
rss1 = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
st = s.stats()
s.step(5)
b = s.stats().loop_seconds
s.step(20)
secs = s.stats().loop_seconds - b
out = {"config": name, "node_order": order, "setup_seconds": round(t_setup, 2), "host_peak_rss_gb": round(rss1, 2),
       "rss_before_gb": round(rss0, 2), "elements": st.n_elems_global, "nodes": st.n_nodes_global,
       "tiles": st.n_tiles, "device_bytes": st.device_bytes, "G_updates_per_s": st.n_elems_global * 20 / secs / 1e9}
if name in ("cfg2", "cfg4") and os.environ.get("COMPARE", "1") == "1":
    Td = s.fields(want_H=False)[0]
    s.close()
    host = configs.CONFIGS[name]()
    with cf.Solver(host.mesh, host.setup, cf.SolveOptions(node_order=order)) as h:
        h.step(25)
        Th = h.fields(want_H=False)[0]
    out["bitwise_vs_host_mesh_plan_25_steps"] = bool(np.array_equal(Td, Th))
print(json.dumps(out), flush=True)
