"""Generates tests/golden/*.npz: nodal temperatures produced by the REFERENCE
solver itself (oracle/_ref, the unmodified castfem headers compiled by
oracle/Makefile) on seeded synthetic cases. Run where /root/reference exists:
    python tests/golden/make_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from test_oracle_pin import CASES  # noqa: E402

STEPS = {"cube6": 40, "casting10": 30, "jitter9_perm": 30, "dirichlet_tdep6": 30, "casting_temp_h": 30}

if __name__ == "__main__":
    for name, steps in STEPS.items():
        m, s = CASES[name]()
        r, _ = orc.ref_solve(m, s, steps)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), case=name, steps=steps, T=r.T, time=r.time,
                            H=r.H, generator="oracle/_ref (reference castfem headers)")
        print(name, m.node_count(), r.time)
