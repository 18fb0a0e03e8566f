"""The RCM reordering pass on the B200 (cf_rcm.cu) against the reference's own rcm_permutation
(reorder.hpp:127-148, oracle/_ref) and the host restatement: the permutation must be equal
element for element -- components by ascending smallest id, George-Liu pseudo-peripheral
roots, per-parent (degree, id) order, explicit seeds, isolated vertices, and vertices whose
degree exceeds the kernel's per-thread neighbour list (its slow path)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf
from paper_1005_3158_b200 import configs
from paper_1005_3158_b200.castfem import _Keep, mesh_desc

pytestmark = pytest.mark.gpu


def ref_rcm(m, seed=-1):
    keep = _Keep()
    d = mesh_desc(m, keep)
    out = np.zeros(m.node_count(), np.int32)
    assert orc.ref_lib().ref_rcm_permutation(C.byref(d), seed, out.ctypes.data_as(C.POINTER(C.c_int32))) == 0
    return out


def _fan(k):
    """k tets sharing node 0 (degree 2k+1 at node 0: beyond the 64-entry fast path), plus an
    isolated node and a separate two-tet component with smaller ids than the fan's far nodes."""
    nodes = [[0.0, 0.0, 0.0]]
    tets = []
    for i in range(k):
        a = len(nodes)
        t = 2 * np.pi * i / k
        nodes += [[np.cos(t), np.sin(t), 0.0], [np.cos(t + 0.1), np.sin(t + 0.1), 0.0], [0.0, 0.0, 1.0 + i]]
        tets.append([0, a, a + 1, a + 2])
    iso = len(nodes)
    nodes.append([9.0, 9.0, 9.0])
    b = len(nodes)
    nodes += [[5, 5, 5], [6, 5, 5], [5, 6, 5], [5, 5, 6], [6, 6, 6]]
    tets += [[b, b + 1, b + 2, b + 3], [b + 1, b + 2, b + 3, b + 4]]
    perm = np.random.default_rng(3).permutation(len(nodes)).astype(np.int32)
    tets = perm[np.array(tets)]
    return cf.Mesh(np.array(nodes)[np.argsort(perm)], tets, np.zeros(len(tets), np.int32), np.zeros((0, 3)),
                   np.zeros(0), []), int(perm[iso])


def _delaunay(n, seed):
    """Unstructured node graph (degrees 4-40, many (degree, id) ties to break)."""
    from scipy.spatial import Delaunay
    pts = np.random.default_rng(seed).random((n, 3))
    tets = Delaunay(pts).simplices.astype(np.int32)
    return cf.Mesh(pts, tets, np.zeros(len(tets), np.int32), np.zeros((0, 3)), np.zeros(0), [])


MESHES = {
    "delaunay800": lambda: _delaunay(800, 31),
    "delaunay3000": lambda: _delaunay(3000, 32),
    "cube5": lambda: cf.generate_fixture("cube", 5),
    "casting9": lambda: cf.generate_fixture("casting", 9),
    "jitter8_perm": lambda: cf.generate_fixture("casting", 8, jitter=0.2, seed=5, perm_seed=17),
    "cube7_perm": lambda: cf.generate_fixture("cube", 7, perm_seed=99),
    "casting24_perm": lambda: cf.generate_fixture("casting", 24, jitter=0.2, seed=2, perm_seed=4),
    "fan40": lambda: _fan(40)[0],
}


@pytest.mark.parametrize("name", sorted(MESHES))
def test_device_rcm_equals_reference(name):
    m = MESHES[name]()
    dev = cf.rcm_permutation_device(m)
    assert np.array_equal(dev, cf.rcm_permutation(m))
    if orc.ref_available():
        assert np.array_equal(dev, ref_rcm(m))
    for seed in (int(m.node_count() // 3), 0, m.node_count() - 1):
        dev_s = cf.rcm_permutation_device(m, seed)
        assert np.array_equal(dev_s, cf.rcm_permutation(m, seed))
        if orc.ref_available():
            assert np.array_equal(dev_s, ref_rcm(m, seed))


def test_device_rcm_isolated_seed():
    m, iso = _fan(70)
    for seed in (iso, -1):
        assert np.array_equal(cf.rcm_permutation_device(m, seed), cf.rcm_permutation(m, seed))


def test_device_rcm_cfg3_equals_host():
    """BASELINE configs[2] (2.06 M tets, jittered, randomly permuted numbering): device == host."""
    m = configs.config3().mesh
    assert np.array_equal(cf.rcm_permutation_device(m), cf.rcm_permutation(m))
