"""Edge cases through the C-ABI on the GPU, each against the CPU oracle
(replaying the GPU's tiles, so deterministic mode must match bit for bit)."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf
from paper_1005_3158_b200 import configs

pytestmark = pytest.mark.gpu


def check(m, s, steps, **kw):
    opts = cf.SolveOptions(max_steps=steps, **kw)
    gpu = cf.solve(m, s, opts)
    tiles, _ = cf.tile_map(m, s, opts)
    ref = orc.solve(m, s, steps, blocks=tiles)
    assert np.array_equal(gpu.T, ref.T), np.abs(gpu.T - ref.T).max()
    assert np.array_equal(gpu.H, ref.H)
    assert gpu.end_time == ref.time and gpu.steps == ref.steps
    return gpu, ref


def test_single_tet_all_faces_convective():
    nodes = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]
    faces = [[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]]
    m = cf.Mesh(nodes, [[0, 1, 2, 3]], [0], faces, [0, 0, 0, 0], ["skin"])
    s = cf.SimulationSetup(materials=[cf.MaterialTable.make(1000.0, 500.0, 10.0, T0=400.0)],
                           boundary_conditions={"skin": cf.BoundaryCondition("flux", q=5.0, h=30.0, t_inf=300.0)},
                           solver=cf.SolverConfig(dt_safety=0.2), initial_T=np.array([400.0, 410.0, 390.0, 405.0]))
    gpu, _ = check(m, s, 25)
    assert np.all(np.diff(gpu.T) != 0)


def test_adiabatic_conservation():
    """No boundary facets: sum_i C_i (T_i' - T_i) = 0, C from the oracle's own lumping."""
    c = configs.config1(n=6)
    m = cf.Mesh(c.mesh.nodes, c.mesh.tets, c.mesh.region, np.zeros((0, 3)), np.zeros(0), [])
    s = cf.SimulationSetup(materials=c.setup.materials, solver=c.setup.solver, initial_T=c.setup.initial_T)
    gpu, _ = check(m, s, 10)
    tets, _ = cf.finalize_mesh(m)
    p = m.nodes[tets]
    V = np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0])) / 6
    Cn = np.zeros(m.node_count())
    np.add.at(Cn, tets.reshape(-1), np.repeat(2700.0 * 900.0 * V / 4, 4))
    assert abs(np.sum(Cn * (gpu.T - s.initial_T))) <= 1e-11 * np.sum(Cn * s.initial_T)


def test_region_gap_and_unused_material_slot():
    c = configs.casting(8, dt_safety=0.14)
    m = c.mesh
    m.region = np.where(m.region == 1, 2, 0).astype(np.int32)          # regions 0 and 2
    mats = [c.setup.materials[0], cf.MaterialTable(), c.setup.materials[1]]  # slot 1 untouched (rho 0)
    s = cf.SimulationSetup(materials=mats, boundary_conditions=c.setup.boundary_conditions,
                           interface_coeffs=c.setup.interface_coeffs, solver=c.setup.solver,
                           initial_T=c.setup.initial_T)
    check(m, s, 20)


def test_two_contacts_and_duplicate_facet_records():
    c = configs.casting(8, dt_safety=0.14)
    m = c.mesh
    # split the interface tags in two halves (x < 0.5 / x >= 0.5): two contact declarations
    cen = m.nodes[m.facets].mean(axis=1)
    tag = m.facet_tag.copy()
    tag[(tag == 1) & (cen[:, 0] >= 0.5)] = 3
    tag[(tag == 2) & (cen[:, 0] >= 0.5)] = 4
    # duplicate the first outer facet record (the reference accumulates it twice)
    first_outer = int(np.where(tag == 0)[0][0])
    facets = np.vstack([m.facets, m.facets[first_outer:first_outer + 1]])
    tag = np.concatenate([tag, [0]]).astype(np.int32)
    m2 = cf.Mesh(m.nodes, m.tets, m.region, facets, tag, ["outer", "cast_if", "mold_if", "cast_if2", "mold_if2"],
                 [(1, 2), (3, 4)])
    s = cf.SimulationSetup(materials=c.setup.materials, boundary_conditions=c.setup.boundary_conditions,
                           interface_coeffs=[c.setup.interface_coeffs[0],
                                             cf.InterfaceCoeff("mold_if2", "cast_if2", "temperature",
                                                               cf.PiecewiseLinear([300.0, 1000.0], [400.0, 3000.0]))],
                           solver=c.setup.solver, initial_T=c.setup.initial_T)
    check(m2, s, 20)
    if orc.ref_available():
        r, _ = orc.ref_solve(m2, s, 20)
        assert np.array_equal(orc.solve(m2, s, 20).T, r.T)


def test_empty_mesh():
    m = cf.Mesh(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0), np.zeros((0, 3)), np.zeros(0), [])
    s = cf.SimulationSetup(materials=[cf.MaterialTable.make(1.0, 1.0, 1.0)], solver=cf.SolverConfig(dt_safety=0.5))
    res = cf.solve(m, s, cf.SolveOptions(max_steps=3))
    assert res.T.shape == (0,) and res.steps == 3


def test_plan_option_validation():
    """Bad run options fail loudly with the C-ABI status, before any device work."""
    import ctypes as C
    from paper_1005_3158_b200 import _abi
    case = configs.casting(6, dt_safety=0.14)
    keep = cf._Keep()
    md, sd = cf.mesh_desc(case.mesh, keep), cf.setup_desc(case.setup, keep)
    for field, value, code in [("fast_math", 1, _abi.CF_CONFIG), ("geometry", 7, _abi.CF_INVALID_ARG),
                               ("mode", 9, _abi.CF_INVALID_ARG), ("tile_elems", 4096, _abi.CF_INVALID_ARG)]:
        ro = cf.run_opts(cf.SolveOptions(), keep)
        setattr(ro, field, value)
        h = C.c_void_p()
        assert _abi.lib().cf_plan_create(C.byref(md), C.byref(sd), C.byref(ro), C.byref(h)) == code, field


def test_nccl_binding_single_rank():
    """The NCCL transport's dlopen'd binding (ncclGetUniqueId / ncclCommInitRank /
    ncclCommDestroy through cf_comm_*) on a one-rank communicator: multi-process runs need
    one GPU per rank, which a one-GPU box cannot host."""
    uid = cf.Comm.unique_id()
    assert len(uid) == 128 and any(uid)
    comm = cf.Comm(1, 0, 0, uid)
    assert comm.handle
    comm.close()
    assert comm.handle is None


@pytest.mark.parametrize("tile_elems", [1, 384])
def test_zero_lumped_capacitance_reported_like_the_reference(tile_elems):
    """explicit_update's error (fem.hpp:110-111): temperatures 1 ulp apart inside the mushy
    range where H absorbs the difference -> |grad H| = 0 while |grad T| > 0 -> Lemmon C_app = 0
    -> c = 0 at every node. The GPU raises the reference's error class and message with the same
    node, from the fused tile-private update (one tile) and from the shared-node update kernel
    (one element per tile)."""
    nodes = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]]
    tets = [[0, 1, 2, 3], [1, 2, 3, 4]]
    faces = [[0, 2, 3], [0, 1, 3], [0, 1, 2], [2, 3, 4], [1, 3, 4], [1, 2, 4]]
    m = cf.Mesh(nodes, tets, [0, 0], faces, [0] * 6, ["skin"])
    T0 = np.full(5, 973.0)
    T0[1] = np.nextafter(973.0, 2000.0)
    mat = cf.MaterialTable.make(2700.0, 900.0, 200.0, latent_heat=3.9e5, solidus=821, liquidus=913, T0=973.0)
    s = cf.SimulationSetup(materials=[mat], boundary_conditions={"skin": cf.BoundaryCondition("flux", h=0.0)},
                           solver=cf.SolverConfig(dt_safety=0.2), initial_T=T0)
    with pytest.raises(orc.OracleError) as ref:
        orc.ref_solve(m, s, 3) if orc.ref_available() else orc.solve(m, s, 3)
    with pytest.raises(cf.ValidationError) as gpu:
        cf.solve(m, s, cf.SolveOptions(max_steps=3, tile_elems=tile_elems))
    assert str(gpu.value) == str(ref.value).split("] ", 1)[1]


def test_atomic_steps_past_t_end_leave_no_stale_sums():
    """Atomic mode (fp64 RED accumulators): steps past t_end are no-ops (solve_serial
    blocked.hpp:674-677) and must not leave partial sums behind for the next real step, nor may
    a re-initialisation (set_temperature). Compared against the deterministic mode (1e-9)."""
    case = configs.casting(10, dt_safety=0.14)
    out = {}
    for mode in ("deterministic", "atomic"):
        with cf.Solver(case.mesh, case.setup, cf.SolveOptions(mode=mode)) as s:
            dt = s.stats().static_dt
            s.step(10, t_end=5.5 * dt)           # 6 real steps (the last one clipped), 4 no-ops
            assert s.stats().step_index == 6
            s.step(8)                            # max_steps mode again
            T1, _ = s.fields(False)
            s.set_temperature(case.setup.initial_T)
            s.step(3, t_end=1.5 * dt)            # 2 real steps, 1 no-op
            s.set_temperature(case.setup.initial_T)
            s.step(5)
            T2, _ = s.fields(False)
            out[mode] = (T1, T2)
    for a, b in zip(out["atomic"], out["deterministic"]):
        assert float(np.max(np.abs(a - b) / np.abs(b))) <= 1e-9


@pytest.mark.parametrize("tile_elems,ranks", [(32, 1), (512, 1), (48, 3)])
def test_high_valence_hub_mesh(tile_elems, ranks):
    """A genuinely unstructured topology: 400 tets fanned around one hub node (the convex hull of
    random points on a sphere, each surface triangle joined to the centre). The hub's reduction
    list holds every element of its tile, and with small tiles the hub is shared by more tiles
    than an update record holds (the merge-list path, > 8 partials) and by every rank."""
    from scipy.spatial import ConvexHull
    rng = np.random.default_rng(5)
    pts = rng.normal(size=(202, 3))
    pts /= np.linalg.norm(pts, axis=1)[:, None]
    pts *= 0.8 + 0.4 * rng.random((202, 1))  # star-shaped, not a sphere: varied element sizes
    hull = ConvexHull(pts / np.linalg.norm(pts, axis=1)[:, None])
    tri = hull.simplices.astype(np.int32) + 1
    nodes = np.vstack([[0.0, 0.0, 0.0], pts])
    tets = np.hstack([np.zeros((len(tri), 1), np.int32), tri])
    m = cf.Mesh(nodes, tets, np.zeros(len(tets), np.int32), tri, np.zeros(len(tri), np.int32), ["outer"])
    mat = cf.MaterialTable.make(rho=2700.0, c=900.0, k=200.0, latent_heat=3.9e5, solidus=821.0, liquidus=913.0,
                                T0=930.0)
    T0 = 930.0 + 20.0 * rng.random(m.node_count())
    s = cf.SimulationSetup(materials=[mat], boundary_conditions={"outer": cf.BoundaryCondition("flux", h=500.0,
                                                                                              t_inf=300.0)},
                           solver=cf.SolverConfig(dt_safety=0.05), initial_T=T0)
    assert len(tets) >= 390
    opts = cf.SolveOptions(max_steps=200, tile_elems=tile_elems, world_size=ranks, local_ranks=ranks)
    gpu = cf.solve(m, s, opts)
    tiles, nt = cf.tile_map(m, s, opts)
    if tile_elems == 32:
        assert nt > 8  # the hub's partial count exceeds an update record
    parts = cf.partition_rcb(m, ranks) if ranks > 1 else None
    ref = orc.solve(m, s, 200, blocks=tiles, parts=parts)
    assert np.array_equal(gpu.T, ref.T), float(np.abs(gpu.T - ref.T).max())
    at = cf.solve(m, s, cf.SolveOptions(max_steps=200, tile_elems=tile_elems, mode="atomic", world_size=ranks,
                                        local_ranks=ranks))
    assert float(np.max(np.abs(at.T - ref.T) / np.abs(ref.T))) <= 1e-9
    assert gpu.T.min() < T0.min()  # it cools


@pytest.mark.parametrize("tile_elems,ranks,geometry", [(128, 1, "stored"), (384, 1, "coords"), (160, 2, "stored")])
def test_delaunay_mesh(tile_elems, ranks, geometry):
    """An unstructured Delaunay tetrahedralisation of 600 random points (3704 tets of every shape,
    slivers included, node valences 5-40; hull faces convective): nothing of the Kuhn fixtures'
    regularity. Deterministic mode bitwise, atomic mode 1e-9, against the oracle on the same tiles
    and parts; dt_safety is small because Eq. 13's bound is not a stability bound on slivers."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(12)
    pts = rng.random((600, 3))
    d = Delaunay(pts)
    tets, hull = d.simplices.astype(np.int32), d.convex_hull.astype(np.int32)
    m = cf.Mesh(pts, tets, np.zeros(len(tets), np.int32), hull, np.zeros(len(hull), np.int32), ["outer"])
    mat = cf.MaterialTable.make(rho=2700.0, c=900.0, k=200.0, latent_heat=3.9e5, solidus=821.0, liquidus=913.0,
                                T0=930.0)
    T0 = 900.0 + 60.0 * rng.random(m.node_count())  # straddles the liquidus: latent heat active
    s = cf.SimulationSetup(materials=[mat], boundary_conditions={"outer": cf.BoundaryCondition("flux", h=500.0,
                                                                                              t_inf=300.0)},
                           solver=cf.SolverConfig(dt_safety=0.01), initial_T=T0)
    steps = 150
    opts = cf.SolveOptions(max_steps=steps, tile_elems=tile_elems, geometry=geometry, world_size=ranks,
                           local_ranks=ranks)
    gpu = cf.solve(m, s, opts)
    tiles, _ = cf.tile_map(m, s, opts)
    parts = cf.partition_rcb(m, ranks) if ranks > 1 else None
    ref = orc.solve(m, s, steps, blocks=tiles, parts=parts)
    assert np.isfinite(ref.T).all() and ref.T.max() < 960.0
    assert np.array_equal(gpu.T, ref.T), float(np.abs(gpu.T - ref.T).max())
    at = cf.solve(m, s, cf.SolveOptions(max_steps=steps, tile_elems=tile_elems, geometry=geometry, mode="atomic",
                                        world_size=ranks, local_ranks=ranks))
    assert float(np.max(np.abs(at.T - ref.T) / np.abs(ref.T))) <= 1e-9
    if orc.ref_available() and ranks == 1:  # and the reference itself, one block
        r, _ = orc.ref_solve(m, s, steps)
        assert float(np.max(np.abs(gpu.T - r.T) / np.abs(r.T))) <= 1e-9


def test_plain_c_caller(tmp_path):
    """tests/c/c_abi_example.c: a C11 program fills the descriptors by hand, creates a plan, steps
    and reads the fields through include/castfem_b200.h alone. Its printed temperatures (hex
    doubles) must equal the oracle's bit for bit in both tile layouts, and a bad facet tag must
    come back as CF_CONFIG with the reference's message."""
    import os
    import subprocess
    from paper_1005_3158_b200 import _abi
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "c_abi_example")
    libdir = os.path.dirname(_abi.LIB_PATH)
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I" + os.path.join(root, "include"),
                        os.path.join(root, "tests", "c", "c_abi_example.c"), "-o", exe, "-L" + libdir, "-lcastfem_b200",
                        "-Wl,-rpath," + libdir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    coords = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 1, 1, 0, 0, 0, 1, 1, 0, 1, 0, 1, 1, 1, 1, 1], float).reshape(8, 3)
    tets = np.array([0, 1, 3, 7, 0, 1, 5, 7, 0, 2, 3, 7, 0, 2, 6, 7, 0, 4, 5, 7, 0, 4, 6, 7], np.int32).reshape(6, 4)
    fac = np.array([0, 1, 3, 0, 2, 3, 4, 5, 7, 4, 6, 7, 0, 1, 5, 0, 4, 5, 2, 3, 7, 2, 6, 7, 0, 2, 6, 0, 4, 6, 1, 3, 7,
                    1, 5, 7], np.int32).reshape(12, 3)
    m = cf.Mesh(coords, tets, np.zeros(6, np.int32), fac, np.zeros(12, np.int32), ["skin"])
    mat = cf.MaterialTable.make(rho=2700.0, c=[(300.0, 850.0), (1000.0, 1100.0)], k=200.0, latent_heat=3.9e5,
                                solidus=821.0, liquidus=913.0, T0=930.0)
    T0 = np.array([930.0, 925.0, 921.5, 917.0, 912.0, 908.5, 903.0, 899.0])
    s = cf.SimulationSetup(materials=[mat], boundary_conditions={"skin": cf.BoundaryCondition("flux", h=50.0,
                                                                                             t_inf=300.0)},
                           solver=cf.SolverConfig(dt_safety=0.002), initial_T=T0)
    lines = out.stdout.strip().splitlines()
    for g, geometry in enumerate(("stored", "coords")):
        opts = cf.SolveOptions(tile_elems=4, geometry=geometry)
        tiles, nt = cf.tile_map(m, s, opts)
        ref = orc.solve(m, s, 25, blocks=tiles)
        head = lines[9 * g].split()
        assert head[:6] == ["geometry", str(g), "steps", "25", "tiles", str(nt)] and nt == 2
        assert float.fromhex(head[7]) == ref.time
        for i in range(8):
            _, idx, t_hex, h_hex = lines[9 * g + 1 + i].split()
            assert int(idx) == i and float.fromhex(t_hex) == ref.T[i] and float.fromhex(h_hex) == ref.H[i]
    assert lines[18] == f"bad tag: status {_abi.CF_CONFIG}: facet tag 'skin' resolves to no declared condition"
