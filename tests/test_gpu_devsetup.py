"""The device setup pipeline (cf_devplan.cu) against the host plan builder (cf_plan.cpp).

The two builders share the per-tile code (cf_tilepack.hpp); everything around it -- finalize,
setup resolution, Morton order and chunking, the shared-memory budget split, local node
numbering, ghosts, merge lists, exchange tables -- is re-implemented with device kernels and
must produce the same plan array for array (cf_plan_digest). The fixture generator on the device
must produce the host fixture, and a plan over it must step bitwise like a plan over the host
mesh. Parity of the stepped results with the oracle is covered by every other GPU test, since
cf_plan_create uses this pipeline by default.
"""
import numpy as np
import pytest

from paper_1005_3158_b200 import castfem as cf
from paper_1005_3158_b200 import configs

pytestmark = pytest.mark.gpu

SKIP = {"tets_ord"}  # not kept by the device pipeline (geometry is computed straight from the mesh)

def _delaunay_case():
    """Unstructured topology (irregular valence, slivers): Delaunay of 500 random points."""
    from types import SimpleNamespace

    from scipy.spatial import Delaunay
    rng = np.random.default_rng(21)
    pts = rng.random((500, 3))
    d = Delaunay(pts)
    tets, hull = d.simplices.astype(np.int32), d.convex_hull.astype(np.int32)
    m = cf.Mesh(pts, tets, np.zeros(len(tets), np.int32), hull, np.zeros(len(hull), np.int32), ["outer"])
    s = cf.SimulationSetup(materials=[cf.MaterialTable.make(rho=2700.0, c=900.0, k=200.0, T0=930.0)],
                           boundary_conditions={"outer": cf.BoundaryCondition("flux", h=500.0, t_inf=300.0)},
                           solver=cf.SolverConfig(dt_safety=0.01))
    return SimpleNamespace(mesh=m, setup=s)


CASES = {
    "delaunay500": _delaunay_case,
    "cast12": lambda: configs.casting(12, dt_safety=0.14),
    "cast16j": lambda: configs.casting(16, jitter=0.2, seed=3, perm_seed=5, dt_safety=0.12),
    "cast24": lambda: configs.casting(24, dt_safety=0.14),
    "cube10": lambda: configs.config1(10),
}
OPTS = [dict(), dict(node_order="tile"), dict(node_order="given"), dict(node_order="rcm"), dict(geometry="coords"),
        dict(elem_order="min_node"), dict(elem_order="given"), dict(tile_elems=256, mode="atomic"),
        dict(world_size=2, rank=1), dict(world_size=3, rank=0, node_order="tile"), dict(world_size=4, rank=3),
        dict(tile_elems=96), dict(tile_elems=768)]


def _key(o):
    return ",".join(f"{k}={v}" for k, v in sorted(o.items())) or "default"


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("opts", OPTS, ids=_key)
def test_device_plan_equals_host_plan(name, opts):
    case = CASES[name]()
    o = cf.SolveOptions(**opts)
    rank = opts.get("rank", 0)
    host = cf.plan_digest(case.mesh, case.setup, o, rank)
    dev = cf.plan_digest(case.mesh, case.setup, o, rank, device=True)
    bad = [k for k in host if k not in SKIP and host[k] != dev[k]]
    assert not bad, f"device plan differs from the host plan in {bad}"


@pytest.mark.parametrize("parts", [2, 3, 4, 8])
def test_device_rcb_equals_host_rcb(parts):
    m = configs.casting(20, jitter=0.2, seed=9, perm_seed=4).mesh
    assert np.array_equal(cf.partition_rcb_device(m, parts), cf.partition_rcb(m, parts))


@pytest.mark.parametrize("env", [{"CF_SLOT_ORDER": "count"}, {"CF_SLOT_BANKS": "0"}, {"CF_BANK_PASSES": "2"},
                                 {"CF_BANK_ITERS": "2"}, {"CF_SMEM_BUDGET": "30000"}], ids=str)
def test_device_plan_builder_knobs(env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    case = configs.casting(16, dt_safety=0.14)
    o = cf.SolveOptions()
    host = cf.plan_digest(case.mesh, case.setup, o)
    dev = cf.plan_digest(case.mesh, case.setup, o, device=True)
    assert all(host[k] == dev[k] for k in host if k not in SKIP)


@pytest.mark.parametrize("name", ["cfg1", "casting20", "casting20j"])
def test_fixture_plan_steps_like_host_mesh_plan(name):
    """A plan over the device-generated fixture (no host mesh) equals a plan over the host
    fixture with the same T0 rule, bit for bit, after 25 steps."""
    if name == "cfg1":
        dc = configs.device_case("cfg1")
        host = configs.config1(32)
    else:
        jit = 0.2 if name.endswith("j") else 0.0
        spec = cf.FixtureSpec("casting", 20, jitter=jit, seed=5, t0_noise=1.0, noise_seed=1)
        dc = configs.DeviceCase(name, spec, configs.casting_setup(0.13), 25)
        host = configs.casting(20, jitter=jit, seed=5, dt_safety=0.13)
    steps = 25
    for mode in ("deterministic", "atomic"):
        o = cf.SolveOptions(max_steps=steps, mode=mode, node_order="rcm")
        with cf.Solver(None, dc.setup, o, fixture=dc.spec) as s:
            st = s.stats()
            assert st.device_setup == 1
            assert st.n_elems_global == host.mesh.element_count() and st.n_nodes_global == host.mesh.node_count()
            T0 = s.fields(want_H=False)[0]
            s.step(steps)
            Td = s.fields(want_H=False)[0]
        assert np.array_equal(T0, host.setup.initial_T)
        ref = cf.solve(host.mesh, host.setup, o)
        if mode == "deterministic":
            assert np.array_equal(Td, ref.T)
        else:
            assert np.max(np.abs(Td - ref.T) / np.abs(ref.T)) <= 1e-9


def test_device_and_host_pipelines_step_identically(monkeypatch):
    case = configs.casting(16, jitter=0.15, seed=2, dt_safety=0.12)
    o = cf.SolveOptions(max_steps=30, node_order="rcm", world_size=2, local_ranks=2)
    dev = cf.solve(case.mesh, case.setup, o)
    monkeypatch.setenv("CF_HOST_SETUP", "1")
    host = cf.solve(case.mesh, case.setup, o)
    assert np.array_equal(dev.T, host.T)


@pytest.mark.parametrize("defect", ["degenerate", "region_conflict", "interior_facet", "bad_index", "no_material"])
def test_device_pipeline_reports_the_host_errors(defect, monkeypatch):
    case = configs.casting(6, dt_safety=0.14)
    m = case.mesh
    if defect == "degenerate":
        m.nodes[m.tets[5, 3]] = m.nodes[m.tets[5, 0]] + 1e-9 * (m.nodes[m.tets[5, 1]] - m.nodes[m.tets[5, 0]])
    elif defect == "region_conflict":
        m.region[7] = 1 - m.region[7]
    elif defect == "interior_facet":
        t = m.tets[0]
        other = np.where((m.tets == t[1]).any(1) & (m.tets == t[2]).any(1) & (m.tets == t[3]).any(1))[0]
        m.facets[0] = t[[1, 2, 3]] if len(other) > 1 else m.facets[0]
    elif defect == "no_material":
        m.region[m.region == 1] = 40  # the mould as region 40: no material (2 declared)
    else:
        m.tets[3, 2] = m.node_count() + 5
    msgs = []
    for host in ("0", "1"):
        monkeypatch.setenv("CF_HOST_SETUP", host)
        with pytest.raises(cf.CastfemError) as ei:
            cf.Solver(m, case.setup, cf.SolveOptions())
        msgs.append((type(ei.value), str(ei.value)))
    assert msgs[0] == msgs[1]


def test_rcm_fixture_is_the_permuted_host_mesh():
    """FixtureSpec(rcm=True): the device fixture renumbered by the device RCM pass equals
    permute_mesh(host fixture, rcm_permutation) -- plan and 20 steps bitwise."""
    spec = cf.FixtureSpec("casting", 18, t0_noise=1.0, noise_seed=1, rcm=True)
    base = configs.casting(18, dt_safety=0.13)
    p = cf.rcm_permutation(base.mesh)
    m = cf.permute_mesh(base.mesh, p)
    T0 = np.empty_like(base.setup.initial_T)
    T0[p] = base.setup.initial_T
    o = cf.SolveOptions(max_steps=20, node_order="tile")
    with cf.Solver(None, configs.casting_setup(0.13), o, fixture=spec) as s:
        assert np.array_equal(s.fields(want_H=False)[0], T0)
        s.step(20)
        Td = s.fields(want_H=False)[0]
    ref = cf.solve(m, configs.casting_setup(0.13, T0=T0), o)
    assert np.array_equal(Td, ref.T)
