"""Product host-side setup (libcastfem_b200.so, CPU only) against the
reference: RCM order (reorder.hpp:127-148), mesh finalize (mesh.hpp:148-207),
sister pairing (mesh.hpp:456-478), exact fixture counts,
RCB partitions, tiling coverage, and the error taxonomy (errors.hpp)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf
from paper_1005_3158_b200 import configs
from paper_1005_3158_b200.castfem import _Keep, mesh_desc

needs_ref = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def _delaunay(n=600, seed=41):
    """Unstructured topology: Delaunay of random points, hull faces as boundary facets."""
    from scipy.spatial import Delaunay
    pts = np.random.default_rng(seed).random((n, 3))
    d = Delaunay(pts)
    tets, hull = d.simplices.astype(np.int32), d.convex_hull.astype(np.int32)
    return cf.Mesh(pts, tets, np.zeros(len(tets), np.int32), hull, np.zeros(len(hull), np.int32), ["outer"])


MESHES = {
    "delaunay600": _delaunay,
    "cube5": lambda: cf.generate_fixture("cube", 5),
    "casting9": lambda: cf.generate_fixture("casting", 9),
    "jitter8_perm": lambda: cf.generate_fixture("casting", 8, jitter=0.2, seed=5, perm_seed=17),
    "cube7_perm": lambda: cf.generate_fixture("cube", 7, perm_seed=99),
}


def ref_call(fn, m, *args):
    keep = _Keep()
    d = mesh_desc(m, keep)
    st = fn(C.byref(d), *args)
    assert st == 0, orc.ref_lib().ref_last_error()


@needs_ref
@pytest.mark.parametrize("name", sorted(MESHES))
def test_rcm_permutation_equals_reference(name):
    m = MESHES[name]()
    ours = cf.rcm_permutation(m)
    ref = np.zeros(m.node_count(), np.int32)
    ref_call(orc.ref_lib().ref_rcm_permutation, m, -1, ref.ctypes.data_as(C.POINTER(C.c_int32)))
    assert np.array_equal(ours, ref)
    seed = int(m.node_count() // 3)
    ours_s = cf.rcm_permutation(m, seed)
    ref_call(orc.ref_lib().ref_rcm_permutation, m, seed, ref.ctypes.data_as(C.POINTER(C.c_int32)))
    assert np.array_equal(ours_s, ref)
    bw = C.c_int64()
    ref_call(orc.ref_lib().ref_bandwidth, m, ours.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(bw))
    assert cf.bandwidth(m, ours) == bw.value  # (RCM can widen structured casting meshes: SURVEY P3)


def test_rcm_kats():
    def path(order):
        nodes = np.array([[i, 0, 0] for i in range(6)], float)
        tets = [[order[0], order[1], order[2], order[3]], [order[1], order[2], order[3], order[4]],
                [order[2], order[3], order[4], order[5]]]
        return cf.Mesh(nodes, tets, [0, 0, 0], np.zeros((0, 3)), np.zeros(0), [])
    m = path([5, 2, 0, 3, 1, 4])
    p = cf.rcm_permutation(m)
    assert sorted(p) == list(range(6))
    assert cf.bandwidth(m, p) <= cf.bandwidth(m)


@needs_ref
@pytest.mark.parametrize("name", sorted(MESHES))
def test_finalize_equals_reference(name):
    m = MESHES[name]()
    tets, owner = cf.finalize_mesh(m)
    rt = np.zeros_like(tets)
    ro = np.zeros(max(1, m.facets.shape[0]), np.int32)
    ref_call(orc.ref_lib().ref_finalize, m, rt.ctypes.data_as(C.POINTER(C.c_int32)),
             ro.ctypes.data_as(C.POINTER(C.c_int32)))
    assert np.array_equal(tets, rt) and np.array_equal(owner, ro[:len(owner)])


@needs_ref
@pytest.mark.parametrize("name", ["casting9", "jitter8_perm"])
def test_sister_pairing_equals_reference(name):
    m = MESHES[name]()
    ours = cf.pair_sister_facets(m)
    n = C.c_int64()
    ref_call(orc.ref_lib().ref_pair_sister_facets, m, None, 0, C.byref(n))
    ref = np.zeros((n.value, 3), np.int32)
    ref_call(orc.ref_lib().ref_pair_sister_facets, m, ref.ctypes.data_as(C.POINTER(C.c_int32)), n.value, C.byref(n))
    assert np.array_equal(ours, ref)
    keep = _Keep()
    d = mesh_desc(m, keep)
    o = np.zeros_like(ref)
    assert orc.oracle_lib().or_pair_sister_facets(C.byref(d), o.ctypes.data_as(C.POINTER(C.c_int32)), n.value,
                                                  C.byref(n)) == 0
    assert np.array_equal(o, ref)


@pytest.mark.parametrize("n,E,N,Fbc,Fif", [
    (32, 196608, 38291, 12288, 9408),
    (70, 2058000, 369169, 58800, 45024),
    (128, 12582912, 2184611, 196608, 151680),
])
def test_fixture_counts_exact(n, E, N, Fbc, Fif):
    """SURVEY §8(d) exact counts (P11), interface nodes duplicated."""
    m = cf.generate_fixture("casting", n, jitter=0.2 if n == 70 else 0.0, seed=7, perm_seed=11 if n == 70 else 0)
    assert m.element_count() == E and m.node_count() == N
    assert int((m.facet_tag == 0).sum()) == Fbc and int((m.facet_tag > 0).sum()) == Fif
    if n == 32:
        cube = cf.generate_fixture("cube", n)
        assert cube.element_count() == 196608 and cube.node_count() == 35937 and cube.facets.shape[0] == 12288


def test_regions_node_disjoint_and_cube_kat():
    m = cf.generate_fixture("cube", 1)  # 6-tet cube, 8 nodes
    assert m.element_count() == 6 and m.node_count() == 8
    c = cf.generate_fixture("casting", 12)
    reg = np.full(c.node_count(), -1)
    for e in range(c.element_count()):
        for n in c.tets[e]:
            assert reg[n] in (-1, c.region[e])
            reg[n] = c.region[e]


def test_rcb_partition_balanced():
    m = cf.generate_fixture("casting", 12)
    for parts in (2, 3, 4, 8):
        p = cf.partition_rcb(m, parts)
        counts = np.bincount(p, minlength=parts)
        assert counts.min() > 0 and counts.max() - counts.min() <= 1


def test_tile_map_covers_every_element_once():
    c = configs.casting(10, dt_safety=0.14)
    for order in ("morton", "min_node", "given"):
        tiles, nt = cf.tile_map(c.mesh, c.setup, cf.SolveOptions(tile_elems=200, elem_order=order))
        assert tiles.min() == 0 and tiles.max() == nt - 1
        assert np.bincount(tiles).max() <= 200


def test_exchange_plan_symmetric():
    c = configs.casting(9, dt_safety=0.14)
    parts = cf.partition_rcb(c.mesh, 3)
    plans = {r: {x["rank"]: x for x in cf.exchange_plan(c.mesh, c.setup, 3, r, parts)} for r in range(3)}
    for r, nb in plans.items():
        for q, x in nb.items():
            y = plans[q][r]
            assert np.array_equal(x["shared"], y["shared"])
            assert np.array_equal(x["ext_to"], y["ext_from"]) and np.array_equal(x["ext_from"], y["ext_to"])
            assert np.all(np.diff(x["shared"]) > 0)


def test_exchange_payload_kat():
    """exchange_and_merge's payload: two workers sharing 3 nodes exchange 6 values
    each way (c and r per shared node), 7 shared nodes 14; the shared lists are ascending and the
    same on both sides."""
    setup = configs.config1(n=1).setup
    s = cf.SimulationSetup(materials=setup.materials, solver=setup.solver)
    none3, none1 = np.zeros((0, 3), np.int32), np.zeros(0, np.int32)
    # two tets glued on one face: 3 shared nodes
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], float)
    m = cf.Mesh(nodes, np.array([[0, 1, 2, 3], [1, 2, 3, 4]], np.int32), np.zeros(2, np.int32), none3, none1, [])
    # a Kuhn cube split 4 + 2 tets shares 6 of its 8 nodes; one more tet of the small part on node 4: 7
    c = cf.generate_fixture("cube", 1)
    nodes7 = np.vstack([c.nodes, [[2.0, 0.0, 0.0], [2.0, 1.0, 0.0], [2.0, 0.0, 1.0]]])
    tets7 = np.vstack([c.tets, [[4, 8, 9, 10]]]).astype(np.int32)
    m7 = cf.Mesh(nodes7, tets7, np.zeros(7, np.int32), none3, none1, [])
    for mesh, parts, n_shared in ((m, [0, 1], 3), (m7, [0, 1, 1, 0, 0, 0, 1], 7)):
        parts = np.array(parts, np.int32)
        a = cf.exchange_plan(mesh, s, 2, 0, parts)
        b = cf.exchange_plan(mesh, s, 2, 1, parts)
        assert len(a) == len(b) == 1 and a[0]["rank"] == 1 and b[0]["rank"] == 0
        assert np.array_equal(a[0]["shared"], b[0]["shared"]) and np.all(np.diff(a[0]["shared"]) > 0)
        assert len(a[0]["shared"]) == n_shared
        for x in (a[0], b[0]):  # no interface facets here: the payload is the (c, r) pairs alone
            assert 2 * len(x["shared"]) + len(x["ext_to"]) == 2 * n_shared


# ---------------------------------------------------------------- error taxonomy
def _tile_status(m, setup):
    try:
        cf.tile_map(m, setup, cf.SolveOptions())
        return 0
    except cf.CastfemError as e:
        return e.code


def test_error_codes():
    c = configs.casting(4, dt_safety=0.14)
    m, s = c.mesh, c.setup
    assert _tile_status(m, s) == 0
    bad = cf.Mesh(m.nodes.copy(), m.tets.copy(), m.region, m.facets, m.facet_tag, m.tags, m.contacts)
    bad.tets[0, 0] = m.node_count() + 5
    assert _tile_status(bad, s) == cf.ValidationError.code                    # dangling node
    deg = cf.Mesh(m.nodes.copy(), m.tets, m.region, m.facets, m.facet_tag, m.tags, m.contacts)
    deg.nodes[deg.tets[3]] = deg.nodes[deg.tets[3][0]] + np.array([[0, 0, 0], [1e-3, 0, 0], [2e-3, 0, 0],
                                                                   [3e-3, 1e-12, 0]])
    assert _tile_status(deg, s) in (cf.DegenerateElementError.code, cf.ValidationError.code)
    s2 = configs.casting(4, dt_safety=0.14).setup
    s2.interface_coeffs = []
    assert _tile_status(m, s2) == cf.ConfigError.code                          # contact without h_i
    s3 = configs.casting(4, dt_safety=0.14).setup
    s3.boundary_conditions = {}
    assert _tile_status(m, s3) == cf.ConfigError.code                          # unresolved tag
    s4 = configs.casting(4, dt_safety=1.5).setup
    assert _tile_status(m, s4) == cf.ConfigError.code                          # safety outside (0, 1]
    s5 = configs.casting(4, dt_safety=0.14).setup
    s5.materials[0].latent_heat = -1.0
    assert _tile_status(m, s5) == cf.ConfigError.code
    shared = cf.Mesh(m.nodes, m.tets.copy(), m.region.copy(), m.facets, m.facet_tag, m.tags, m.contacts)
    shared.region[0] = 1 - shared.region[0]                                    # regions share a node
    assert _tile_status(shared, s) == cf.ValidationError.code


# ---------------------------------------------------------------- tile autotuner (host parts)
def test_choose_tile_elems_semantics():
    """choose_block_count (blocked.hpp:566-575): argmin, the first candidate wins ties; a
    timing per candidate is required."""
    assert cf.choose_tile_elems([192, 384, 768], [3.0, 1.0, 2.0]) == 384
    assert cf.choose_tile_elems([192, 384, 768], [1.0, 1.0, 0.5 + 0.5]) == 192
    assert cf.choose_tile_elems([384, 768], [float("inf"), 2.0]) == 768
    with pytest.raises(cf.ValidationError):
        cf.choose_tile_elems([192, 384], [1.0])
    with pytest.raises(cf.ValidationError):
        cf.choose_tile_elems([], [])


def test_default_tile_candidates():
    assert cf.default_tile_candidates(12_582_912) == [192, 384, 768, 1536]
    assert cf.default_tile_candidates(100_000) == [192, 384]   # >= 148 tiles each
    assert cf.default_tile_candidates(1_000) == [192]          # always one candidate


# ---------------------------------------------------------------- graph partitioning
PART_MESHES = {
    "casting8": lambda: cf.generate_fixture("casting", 8),
    "jitter7_perm": lambda: cf.generate_fixture("casting", 7, jitter=0.2, seed=5, perm_seed=17),
    "cube5_perm": lambda: cf.generate_fixture("cube", 5, perm_seed=3),
    "delaunay400": lambda: _delaunay(400, 43),
}


@needs_ref
@pytest.mark.parametrize("name", sorted(PART_MESHES))
@pytest.mark.parametrize("k,augment", [(2, True), (3, True), (5, False), (8, True)])
def test_graph_partition_equals_reference(name, k, augment):
    """partition_graph over the (virtual-element augmented) dual graph: the same part of every
    element as the reference's partition_elements / partition_graph, and the same quality."""
    m = PART_MESHES[name]()
    ours = cf.partition_elements(m, k, 0.05, augment)
    ref = np.zeros(m.element_count(), np.int32)
    ref_call(orc.ref_lib().ref_partition, m, k, 0.05, int(augment), ref.ctypes.data_as(C.POINTER(C.c_int32)))
    assert np.array_equal(ours, ref)
    q = cf.partition_metrics(m, ours, k)
    cut, split, imb = C.c_int64(), C.c_int64(), C.c_double()
    nb = np.zeros(k, np.int32)
    ref_call(orc.ref_lib().ref_partition_metrics, m, ours.ctypes.data_as(C.POINTER(C.c_int32)), k, C.byref(cut),
             C.byref(imb), nb.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(split))
    assert (q.edge_cut, q.imbalance, q.neighbor_counts, q.split_interface_pairs) == \
        (cut.value, imb.value, nb.tolist(), split.value)


def test_virtual_elements_keep_interface_pairs_together():
    """The point of the augmentation (paper 4.1.1): fewer interface pairs split across parts."""
    m = cf.generate_fixture("casting", 10)
    plain = cf.partition_metrics(m, cf.partition_elements(m, 4, augment=False), 4)
    aug = cf.partition_metrics(m, cf.partition_elements(m, 4, augment=True), 4)
    assert aug.split_interface_pairs < plain.split_interface_pairs
    assert aug.imbalance <= 1.06


def test_partition_errors_like_reference():
    m = cf.generate_fixture("cube", 2)
    with pytest.raises(cf.ValidationError, match="requested 100 parts for 48 weighted elements"):
        cf.partition_elements(m, 100)
    with pytest.raises(cf.ValidationError):
        cf.partition_metrics(m, np.full(m.element_count(), 7, np.int32), 2)


def test_plan_digests_golden():
    """The host plan builder (and with it the per-tile code shared with the device builder)
    reproduces the committed plan digests (tests/golden/make_plan_digests.py)."""
    import json
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from make_plan_digests import digests
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "plan_digests.json")) as f:
        want = json.load(f)
    got = digests()
    assert got.keys() == want.keys()
    bad = [(k, a) for k in want for a in want[k] if want[k][a] != got[k][a]]
    assert not bad, bad[:5]


def test_device_case_specs_match_host_cases():
    """configs.device_case: the same fixture rule and physics as the host-built cases (the mesh
    itself is compared on the GPU, tests/test_gpu_devsetup.py)."""
    from paper_1005_3158_b200 import configs
    for name in ("cfg2", "cfg4", "cfg5"):
        dc = configs.device_case(name)
        assert dc.spec.kind == "casting" and dc.spec.radius == 0.35 and dc.spec.t0_noise == configs.T0_NOISE
        assert dc.setup.solver.dt_safety == configs.DT_SAFETY[name] and dc.setup.initial_T is None
        assert dc.spec.rcm == (name == "cfg2")
        d = dc.spec.desc()
        assert (d.kind, d.n, d.perm_seed, d.rcm) == (1, dc.spec.n, 0, int(dc.spec.rcm))
    assert configs.device_case("cfg1").spec.kind == "cube"
    with pytest.raises(cf.InvalidArgument):
        cf.Solver(None, configs.device_case("cfg2").setup)
