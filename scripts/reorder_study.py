"""BASELINE configs[2]: 70^3 jittered casting with randomly permuted element and
node numbering, run "both unordered and RCM-reordered to measure the
reordering effect" — on the B200 path (three orderings) and with the
reference CPU solver (unordered vs RCM-renumbered + element-sorted mesh)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402

out = {"config": "cfg3: 70^3 cells, 2,058,000 tets, jitter 0.2h, random element+node permutation"}
case = configs.config3()
m, s = case.mesh, case.setup
E = m.element_count()
ref_T = None
for name, no, eo in [("unordered (given nodes, given elements)", "given", "given"),
                     ("RCM nodes + element sort by min RCM label (paper's cache blocks)", "rcm", "min_node"),
                     ("tile first-touch nodes + Morton elements (default)", "tile", "morton")]:
    t0 = time.time()
    with cf.Solver(m, s, cf.SolveOptions(node_order=no, elem_order=eo)) as sv:
        setup_s = time.time() - t0
        sv.step(5)
        ph = sv.time_phases(50)
        before = sv.stats().loop_seconds
        sv.step(200)
        secs = sv.stats().loop_seconds - before
        T, _ = sv.fields(False)
    if ref_T is None:
        ref_T = T
    out[name] = {"ms_per_step": 1e3 * secs / 200, "element_updates_per_s": E * 200 / secs,
                 "tile_kernel_ms": ph[0], "update_kernel_ms": ph[3], "setup_s": setup_s,
                 "max_rel_vs_unordered": float(np.max(np.abs(T - ref_T) / np.abs(ref_T)))}
    print(name, out[name], flush=True)

# reference CPU solver: unordered vs RCM-permuted nodes + elements sorted by min node label
try:
    from oracle import oracle as orc
    if orc.ref_available():
        perm = cf.rcm_permutation(m)
        mp = cf.permute_mesh(m, perm)
        key = mp.tets.min(axis=1)
        order = np.argsort(key, kind="stable")
        mp = cf.Mesh(mp.nodes, mp.tets[order], mp.region[order], mp.facets, mp.facet_tag, mp.tags, mp.contacts,
                     mp.node_grid)
        sp = configs.config3().setup
        sp.initial_T = s.initial_T[np.argsort(perm)] if s.initial_T is not None else None
        # permute_mesh: new_of_old -> node new index p[i] holds old node i
        T0new = np.empty_like(s.initial_T)
        T0new[perm] = s.initial_T
        sp.initial_T = T0new
        for label, mm, ss in [("reference unordered", m, s), ("reference RCM + element sort", mp, sp)]:
            rb = orc.RefBench(mm, ss)
            rb.steps(1)
            secs = rb.steps(5)
            rb.close()
            out[label] = {"ns_per_tet_step": 1e9 * secs / (5 * E), "element_updates_per_s": 5 * E / secs, "cores": 1}
            print(label, out[label], flush=True)
        out["bandwidth_given"] = cf.bandwidth(m)
        out["bandwidth_rcm"] = cf.bandwidth(m, perm)
except Exception as e:  # report, do not fail the study
    out["reference_error"] = str(e)
print(json.dumps(out))
