"""Times the device RCM pass (cf_rcm.cu) on a BASELINE mesh: python scripts/time_rcm.py cfg5"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
m = configs.CONFIGS[name]().mesh
t0 = time.time()
p = cf.rcm_permutation_device(m)
t1 = time.time()
print(f"{name}: N={m.node_count()} E={m.element_count()} device RCM {t1 - t0:.2f} s")
if m.node_count() < 5_000_000:
    h = cf.rcm_permutation(m)
    print(f"host RCM {time.time() - t1:.2f} s, equal: {bool((h == p).all())}")
