"""The CPU oracle (oracle/castfem_oracle.c, a C restatement) against the
reference itself (oracle/_ref: the unmodified castfem headers) — bitwise —
and against the SPEC known-answer examples. With /root/reference absent the
committed golden vectors (tests/golden/, made by tests/golden/make_golden.py
from the reference) pin it instead."""
import ctypes as C
import glob
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf
from paper_1005_3158_b200 import configs

HERE = os.path.dirname(os.path.abspath(__file__))
needs_ref = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
_dp = C.POINTER(C.c_double)


def dirichlet_case(n=6):
    m = cf.generate_fixture("cube", n)
    x0 = np.all(m.nodes[m.facets][:, :, 0] == 0.0, axis=1)
    m.facet_tag = np.where(x0, 1, 0).astype(np.int32)
    m.tags = ["outer", "hot"]
    mat = cf.MaterialTable.make(rho=7800.0, c=[(300.0, 450.0), (900.0, 700.0)], k=[(300.0, 45.0), (900.0, 30.0)],
                                latent_heat=2.0e5, solidus=700.0, liquidus=760.0, T0=650.0)
    setup = cf.SimulationSetup(
        materials=[mat],
        boundary_conditions={"outer": cf.BoundaryCondition("flux", h=50.0, t_inf=300.0),
                             "hot": cf.BoundaryCondition("fixed", fixed_T=cf.PiecewiseLinear([0.0, 50.0],
                                                                                          [650.0, 950.0]))},
        solver=cf.SolverConfig(dt_safety=0.1))
    return m, setup


CASES = {
    "cube6": lambda: (lambda c: (c.mesh, c.setup))(configs.config1(n=6)),
    "casting10": lambda: (lambda c: (c.mesh, c.setup))(configs.casting(10, dt_safety=0.14)),
    "jitter9_perm": lambda: (lambda c: (c.mesh, c.setup))(configs.casting(9, jitter=0.2, seed=4, perm_seed=3,
                                                                          dt_safety=0.14)),
    "dirichlet_tdep6": dirichlet_case,
    "casting_temp_h": lambda: _temp_h_case(),
}


def _temp_h_case():
    c = configs.casting(8, dt_safety=0.14)
    c.setup.interface_coeffs[0] = cf.InterfaceCoeff("cast_if", "mold_if", "temperature",
                                                    cf.PiecewiseLinear([300.0, 900.0], [500.0, 2000.0]))
    return c.mesh, c.setup


@needs_ref
@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_bitwise_equals_reference(name):
    m, s = CASES[name]()
    o = orc.solve(m, s, 25)
    r, _ = orc.ref_solve(m, s, 25)
    assert np.array_equal(o.T, r.T), np.abs(o.T - r.T).max()
    assert np.array_equal(o.H, r.H)
    assert o.time == r.time and o.steps == r.steps and o.clamp_steps == r.clamp_steps


@needs_ref
@pytest.mark.parametrize("blocks", [3, 8])
def test_oracle_replays_reference_blocks(blocks):
    """BlockPlan semantics: the oracle fed the reference's own partition_graph
    blocks reproduces the reference's blocked run bit for bit."""
    c = configs.casting(9, dt_safety=0.14)
    r, bm = orc.ref_solve(c.mesh, c.setup, 20, blocks=blocks)
    o = orc.solve(c.mesh, c.setup, 20, blocks=bm)
    assert np.array_equal(o.T, r.T)
    one = orc.solve(c.mesh, c.setup, 20)
    assert np.max(np.abs(o.T - one.T) / one.T) < 1e-14  # block-count independence


@needs_ref
def test_t_end_mode_and_series_match_reference():
    c = configs.casting(8, dt_safety=0.14)
    c.setup.solver.output_every = 4
    c.setup.solver.t_end = 10.3 * orc.solve(c.mesh, c.setup, 1).dt
    o = orc.solve(c.mesh, c.setup, 0)
    r, _ = orc.ref_solve(c.mesh, c.setup, 0)
    assert o.steps == r.steps == 11 and o.time == r.time
    assert np.array_equal(o.T, r.T) and np.array_equal(o.series, r.series)


def test_oracle_matches_golden_vectors():
    files = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))
    assert files, "tests/golden is empty: run tests/golden/make_golden.py"
    for f in files:
        g = np.load(f)
        m, s = CASES[str(g["case"])]()
        o = orc.solve(m, s, int(g["steps"]))
        assert np.array_equal(o.T, g["T"]), f
        assert o.time == float(g["time"])


# ---------------------------------------------------------------- SPEC known answers
def _geom(p):
    out = np.zeros(15)
    st = orc.oracle_lib().or_tet_geometry(np.ascontiguousarray(p, dtype=np.float64).ctypes.data_as(_dp),
                                          out.ctypes.data_as(_dp))
    return st, out


def test_kat_tet_geometry_unit_tet():
    st, g = _geom([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1])
    assert st == 0 and g[0] == 1.0 / 6.0
    assert np.array_equal(g[1:13].reshape(4, 3), [[-1, -1, -1], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    st, _ = _geom([0, 0, 0, 1, 0, 0, 2, 0, 0, 0, 0, 1e-9])
    assert st == 5  # degenerate (CF_DEGENERATE)


def test_kat_geometry_partition_of_unity_and_linear_field():
    rng = np.random.default_rng(3)
    for _ in range(20):
        p = rng.normal(size=(4, 3))
        if np.linalg.det(p[1:] - p[0]) < 0:
            p[[2, 3]] = p[[3, 2]]
        st, g = _geom(p.reshape(-1))
        grads = g[1:13].reshape(4, 3)
        assert np.abs(grads.sum(0)).max() < 1e-12 * np.abs(grads).max()
        assert np.allclose(grads.T @ p[:, 0], [1, 0, 0], atol=1e-9)  # grad of T = x


def _mat(c=1.0, L=0.0, ts=0.0, tl=1.0, rho=1.0, k=1.0):
    from paper_1005_3158_b200.castfem import _Keep, _abi
    keep = _Keep()
    m = cf.MaterialTable.make(rho=rho, c=c, k=k, latent_heat=L, solidus=ts, liquidus=tl)
    return _abi.cf_material(m.rho, keep.table(m.c_of_T), keep.table(m.k_of_T), m.latent_heat, m.solidus, m.liquidus,
                            0.0), keep


def test_kat_enthalpy():
    m, keep = _mat(c=2.0)
    assert orc.oracle_lib().or_enthalpy(C.byref(m), 3.0) == 6.0
    m, keep = _mat(c=1.0, L=100.0, ts=0.0, tl=1.0)
    assert orc.oracle_lib().or_enthalpy(C.byref(m), 1.0) == 101.0
    xs = np.sort(np.random.default_rng(0).uniform(-2, 3, 1000))
    hs = [orc.oracle_lib().or_enthalpy(C.byref(m), float(x)) for x in xs]
    assert np.all(np.diff(hs) >= 0)


def test_kat_apparent_heat_capacity():
    _, g = _geom([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1])
    gp = g.ctypes.data_as(_dp)
    m, keep = _mat(c=7.0)
    T = np.array([1.0, 2.0, 4.0, 3.0])
    H = 2.0 * T + 5.0
    f = orc.oracle_lib().or_apparent_heat_capacity
    assert f(gp, T.ctypes.data_as(_dp), H.ctypes.data_as(_dp), C.byref(m)) == 2.0
    Tu = np.full(4, 5.0)
    assert f(gp, Tu.ctypes.data_as(_dp), Tu.ctypes.data_as(_dp), C.byref(m)) == 7.0  # c(T bar)
    m2, keep2 = _mat(c=1.0, L=100.0, ts=0.0, tl=1.0)
    T2 = np.array([0.0, 1.0, 0.0, 0.0])
    H2 = np.array([orc.oracle_lib().or_enthalpy(C.byref(m2), t) for t in T2])
    grads = g[1:13].reshape(4, 3)
    brute = np.sqrt(np.sum((grads.T @ H2) ** 2) / np.sum((grads.T @ T2) ** 2))
    assert abs(f(gp, T2.ctypes.data_as(_dp), H2.ctypes.data_as(_dp), C.byref(m2)) - brute) < 1e-12 * brute


def test_kat_assemble_local():
    _, g = _geom([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1])
    m, keep = _mat(c=1.0)
    T = np.full(4, 3.0)
    c = np.zeros(4)
    r = np.zeros(4)
    orc.oracle_lib().or_element_accumulate(g.ctypes.data_as(_dp), C.byref(m), T.ctypes.data_as(_dp),
                                           T.ctypes.data_as(_dp), c.ctypes.data_as(_dp), r.ctypes.data_as(_dp))
    assert np.all(r == 0.0)            # uniform T -> zero residual
    assert np.allclose(c, 1.0 / 24.0)  # rho C = 1, V = 1/6 -> V/4


@needs_ref
def test_kats_agree_with_reference_functions():
    rng = np.random.default_rng(9)
    m, keep = _mat(c=900.0, L=3.9e5, ts=821.0, tl=913.0, rho=2700.0, k=200.0)
    for _ in range(200):
        p = rng.normal(size=12)
        go = np.zeros(15)
        gr = np.zeros(15)
        so = orc.oracle_lib().or_tet_geometry(p.ctypes.data_as(_dp), go.ctypes.data_as(_dp))
        sr = orc.ref_lib().ref_tet_geometry(p.ctypes.data_as(_dp), gr.ctypes.data_as(_dp))
        assert so == sr
        if so:
            continue
        assert np.array_equal(go, gr)
        T = rng.uniform(800, 930, 4)
        H = np.array([orc.oracle_lib().or_enthalpy(C.byref(m), t) for t in T])
        Hr = np.array([orc.ref_lib().ref_enthalpy(C.byref(m), t) for t in T])
        assert np.array_equal(H, Hr)
        a = orc.oracle_lib().or_apparent_heat_capacity(go.ctypes.data_as(_dp), T.ctypes.data_as(_dp),
                                                       H.ctypes.data_as(_dp), C.byref(m))
        b = orc.ref_lib().ref_apparent_heat_capacity(go.ctypes.data_as(_dp), T.ctypes.data_as(_dp),
                                                     H.ctypes.data_as(_dp), C.byref(m))
        assert a == b


def test_kat_stable_timestep():  # rho=c=k=1, l=0.1 -> 0.01 (x safety)
    h = 0.1
    nodes = np.array([[0, 0, 0], [h, 0, 0], [0, h, 0], [0, 0, h]], float)
    m = cf.Mesh(nodes, [[0, 1, 2, 3]], [0], np.zeros((0, 3)), np.zeros(0), [])
    s = cf.SimulationSetup(materials=[cf.MaterialTable.make(1.0, 1.0, 1.0, T0=1.0)],
                           solver=cf.SolverConfig(dt_safety=1.0))
    assert abs(orc.solve(m, s, 1).static_dt - 0.01) < 1e-17
    s.solver.dt_safety = 0.5
    assert abs(orc.solve(m, s, 1).static_dt - 0.005) < 1e-17


def test_kat_conservation_adiabatic():  # sum C (T' - T) = 0, no boundary facets
    c = configs.config1(n=4)
    c.mesh.facets = np.zeros((0, 3), np.int32)
    c.mesh.facet_tag = np.zeros(0, np.int32)
    c.setup.boundary_conditions = {}
    T0 = c.setup.initial_T
    o = orc.solve(c.mesh, c.setup, 1)
    tets, _ = cf.finalize_mesh(c.mesh)
    p = c.mesh.nodes[tets]
    V = np.abs(np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]))) / 6
    Cn = np.zeros(c.mesh.node_count())
    np.add.at(Cn, tets.reshape(-1), np.repeat(2700.0 * 900.0 * V / 4, 4))
    assert abs(np.sum(Cn * (o.T - T0))) <= 1e-12 * np.sum(Cn * T0)


# ---------------------------------------------------------------- the reference arm's own workload generator
@pytest.mark.parametrize("kind,n,radius,jitter,seed,perm", [("cube", 5, 0.35, 0.0, 0, 0), ("casting", 8, 0.35, 0.0, 0, 0),
                                                            ("casting", 9, 0.35, 0.2, 3, 5),
                                                            ("casting", 10, 0.3, 0.1, 2, 0)])
def test_oracle_fixture_generator_equals_product(kind, n, radius, jitter, seed, perm):
    """oracle/fixture.c (used by the reference arm, which must not load the product library)
    reproduces the product's cf_generate_fixture bit for bit, including the non-integer
    radius path, jitter keys and the node / element permutations; a full window is the mesh."""
    p = cf.generate_fixture(kind, n, radius=radius, jitter=jitter, seed=seed, perm_seed=perm)
    for window in (None, [0, n, 0, n, 0, n]):
        o = orc.generate_fixture(kind, n, radius, jitter, seed, perm, window=window)
        assert np.array_equal(o["nodes"], p.nodes)
        assert np.array_equal(o["tets"], p.tets) and np.array_equal(o["region"], p.region)
        assert np.array_equal(o["facets"], p.facets) and np.array_equal(o["facet_tag"], p.facet_tag)
        assert np.array_equal(o["node_grid"], p.node_grid)
    keys = np.arange(1000, dtype=np.int64) * 7919
    assert np.array_equal(orc.counter_uniform(1, keys, -1.0, 1.0), cf.counter_uniform(1, keys, -1.0, 1.0))


def test_oracle_fixture_window_is_a_box_of_the_mesh():
    """A window keeps the full mesh's coordinates, regions and global grid keys; facets only on
    the box boundary and the cast/mould interface (cut planes are adiabatic)."""
    n, w = 16, [2, 14, 0, 16, 5, 9]
    full = orc.generate_fixture("casting", n, jitter=0.2, seed=3)
    win = orc.generate_fixture("casting", n, jitter=0.2, seed=3, window=w)
    cells = (w[1] - w[0]) * (w[3] - w[2]) * (w[5] - w[4])
    assert win["tets"].shape[0] == 6 * cells
    P = n + 1
    g = win["node_grid"]
    gi, gj, gk = g % P, (g // P) % P, g // (P * P)
    assert gi.min() == w[0] and gi.max() == w[1] and gk.min() == w[4] and gk.max() == w[5]
    pos = {int(a): full["nodes"][i] for i, a in enumerate(full["node_grid"])}
    assert all(np.array_equal(win["nodes"][i], pos[int(g[i])]) for i in range(0, len(g), 37))
    fx = win["nodes"][win["facets"]]  # (F, 3, 3)
    outer = win["facet_tag"] == 0
    on_box = np.any(np.all(np.isclose(fx, 0.0) | np.isclose(fx, 1.0), axis=1), axis=1)
    assert on_box[outer].all()
    assert np.bincount(win["facet_tag"], minlength=3)[1] == np.bincount(win["facet_tag"], minlength=3)[2]


@needs_ref
def test_ref_bench_workloads_equal_the_product_configs():
    """oracle/_ref/ref_bench (the reference arm) builds BASELINE's workloads exactly like
    paper_1005_3158_b200/configs.py: same mesh counts, dt_safety, h_i and initial field."""
    for name in ("cfg1", "cfg2", "cfg3"):
        d = orc.ref_bench(name, describe=True)
        case = configs.CONFIGS[name]()
        assert d["elements"] == case.mesh.element_count() and d["nodes"] == case.mesh.node_count()
        assert d["facets"] == case.mesh.facets.shape[0]
        assert d["dt_safety"] == case.setup.solver.dt_safety == configs.DT_SAFETY[name]
        assert d["h_interface"] == configs.H_INTERFACE
        assert d["T0_sum"] == float(np.cumsum(case.setup.initial_T)[-1])
    for name in ("cfg4", "cfg5"):  # too large to generate here: the constants
        d = orc.ref_bench(name, describe=True, window=[0, 8, 0, 8, 0, 8])
        assert d["dt_safety"] == configs.DT_SAFETY[name]


@needs_ref
def test_ref_bench_steps_equal_reference_solve(tmp_path):
    """The reference arm's timed loop is the reference solver: 5 steps of cfg1 and of a 24^3
    casting window through ref_bench equal ref_solve on the product-generated mesh bit for bit."""
    dump = str(tmp_path / "T.bin")
    orc.ref_bench("cfg1", steps=4, warmup=1, dump_T=dump)
    case = configs.config1()
    r, _ = orc.ref_solve(case.mesh, case.setup, 5)
    assert np.array_equal(np.fromfile(dump), r.T)
