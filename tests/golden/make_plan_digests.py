"""Regenerates tests/golden/plan_digests.json: per-array digests of the HOST plan builder
(cf_plan_digest) on two meshes x six option sets. Regression guard for the per-tile code shared
with the device builder (cf_tilepack.hpp): a deliberate change to the tile layout or ordering
regenerates this file; an accidental one fails tests/test_host.py::test_plan_digests_golden.
The digests were first taken from the builder that the GPU parity suite had validated bitwise
against the oracle (round 2, before the device builder existed)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1005_3158_b200 import castfem as cf  # noqa: E402
from paper_1005_3158_b200 import configs  # noqa: E402

CASES = {"cast12": lambda: configs.casting(12, dt_safety=0.14),
         "cast16j": lambda: configs.casting(16, jitter=0.2, seed=3, perm_seed=5, dt_safety=0.12)}
OPTS = [dict(), dict(node_order="tile"), dict(geometry="coords"), dict(elem_order="min_node"),
        dict(world_size=3, rank=1), dict(tile_elems=96)]


def digests():
    out = {}
    for n, f in CASES.items():
        c = f()
        for o in OPTS:
            k = n + ":" + (",".join(f"{a}={b}" for a, b in sorted(o.items())) or "default")
            d = cf.plan_digest(c.mesh, c.setup, cf.SolveOptions(**o), o.get("rank", 0))
            out[k] = {a: format(b, "016x") for a, b in d.items()}
    return out


if __name__ == "__main__":
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "plan_digests.json"), "w") as f:
        json.dump(digests(), f, indent=1, sort_keys=True)
