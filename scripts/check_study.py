"""Diagnostics: the reorder-study Solver flow vs cf.solve for the same steps, cfg3 orderings."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
case = configs.config3()
m, s = case.mesh, case.setup
res = {}
for no, eo in [("given", "given"), ("tile", "morton")]:
    with cf.Solver(m, s, cf.SolveOptions(node_order=no, elem_order=eo)) as sv:
        sv.step(5)
        sv.time_phases(50)
        sv.step(200)
        T, _ = sv.fields(False)
        st = sv.stats()
    r = cf.solve(m, s, cf.SolveOptions(max_steps=255, node_order=no, elem_order=eo))
    res[eo] = (T, r.T)
    print(eo, "steps", st.step_index, "flow vs solve bitwise", np.array_equal(T, r.T), "differing", int(np.sum(T != r.T)), flush=True)
print("flow: morton vs given differing", int(np.sum(res["morton"][0] != res["given"][0])))
print("solve: morton vs given differing", int(np.sum(res["morton"][1] != res["given"][1])))
