import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1005_3158_b200 import castfem as cf, configs
from oracle import oracle as orc
case = configs.config2()
for mode in ["atomic", "deterministic"]:
    s = cf.Solver(case.mesh, case.setup, cf.SolveOptions(mode=mode))
    t = time.time()
    for k in range(10):
        s.step(100)
        T, _ = s.fields(False)
        print(mode, (k + 1) * 100, T.min(), T.max(), "mushy", int(((T > 821) & (T < 913)).sum()), flush=True)
    print(mode, "wall", time.time() - t, "loop", s.stats().loop_seconds)
    s.close()
s = cf.Solver(case.mesh, case.setup, cf.SolveOptions(mode="atomic"))
rb = orc.RefBench(case.mesh, case.setup)
s.step(40); rb.steps(40)
T, _ = s.fields(False); To = rb.T()
print("40 steps gpu vs reference rel", np.max(np.abs(T - To) / np.abs(To)))
