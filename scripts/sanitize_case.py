"""Small end-to-end run for compute-sanitizer (scripts/sanitize.sh): a 12^3 casting (phase
change, interface facets with the lagged ambient, convective BCs), both tile layouts, both
modes, a 2-rank in-process decomposition, and the device RCM pass; 3 steps each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402

case = configs.casting(12, jitter=0.1, seed=3, dt_safety=0.14)
for geometry in ("stored", "coords"):
    for mode in ("deterministic", "atomic"):
        cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=3, mode=mode, geometry=geometry, tile_elems=256))
cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=3, world_size=2, local_ranks=2, tile_elems=256))
cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=3, node_order="rcm"))
print("sanitize case done")
