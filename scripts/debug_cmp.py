import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
from oracle import oracle as orc
n = int(sys.argv[1]); mode = sys.argv[2]; node = int(sys.argv[3])
case = configs.config2(n)
s = cf.Solver(case.mesh, case.setup, cf.SolveOptions(mode=mode))
rb = orc.RefBench(case.mesh, case.setup)
m = case.mesh
print("node", node, "pos", m.nodes[node], "grid", m.node_grid[node], "elems", np.where((m.tets == node).any(1))[0][:30])
for k in range(1, 41):
    try:
        s.step(1)
    except Exception as e:
        print("step", k, "FAIL", e); 
        rb.steps(1); To = rb.T(); print("oracle T node", To[node]); break
    rb.steps(1)
    T, _ = s.fields(False); To = rb.T()
    d = np.abs(T - To) / np.abs(To)
    print(k, "rel", d.max(), "argmax", d.argmax(), "T[node]", T[node], To[node], flush=True)
