import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
from oracle import oracle as orc
n = int(sys.argv[1]); steps = int(sys.argv[2]); every = int(sys.argv[3])
case = configs.config2(n)
s = cf.Solver(case.mesh, case.setup, cf.SolveOptions(mode=sys.argv[4]))
for k in range(0, steps, every):
    try:
        s.step(every)
    except Exception as e:
        print("step", k, "FAIL", e); break
    T, _ = s.fields(False)
    i = np.argmax(np.abs(T - 600))
    print(k + every, T.min(), T.max(), "worst node", i, T[i], flush=True)
if n <= 40:
    o = orc.solve(case.mesh, case.setup, steps)
    T, _ = s.fields(False)
    print("oracle minmax", o.T.min(), o.T.max(), "rel", np.max(np.abs(T - o.T) / np.abs(o.T)))
