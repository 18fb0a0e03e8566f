"""Parity at BASELINE.json's configurations as specified.

Every comparison is against the CPU checkers: the oracle replaying the GPU's own tiles (bitwise
in deterministic mode: same summation order) and the oracle / the reference itself with one
block (<= 1e-9 relative, north_star: only the summation order differs). The CPU runs proceed
concurrently in threads (ctypes releases the GIL), so the suite stays within minutes.

  cfg2  128^3 casting, 12.6 M tets, RCM-reordered as configs[1] states and the default order:
        100 steps; the full 1000 steps run once as a slow job (scripts/cfg2_full_parity.py,
        profiles/r02_cfg2_full_parity.json).
  cfg3  70^3 jittered casting, randomly permuted numbering, 500 steps, all three orderings.
  cfg4  256^3 casting (100.7 M tets): 3 steps against the reference solver itself.
  cfg5  512^3 casting (805 M tets, one B200): 2 steps against the oracle on a z-slab window of
        the same mesh, compared at nodes >= 4 cells from the window's cut planes (an explicit
        step couples only nodes that share an element, so 2 steps cannot carry the cut's
        influence that far).
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf
from paper_1005_3158_b200 import configs

pytestmark = pytest.mark.gpu
RTOL = 1e-9


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


def ref_steps(mesh, setup, steps):
    rb = orc.RefBench(mesh, setup)
    try:
        rb.steps(steps)
        return rb.T()
    finally:
        rb.close()


def test_cfg2_rcm_and_default_orders_100_steps():
    case = configs.config2()
    steps = 100
    out, tiles = {}, {}
    for order in ("rcm", "tile"):
        opts = cf.SolveOptions(max_steps=steps, node_order=order)
        r = cf.solve(case.mesh, case.setup, opts)
        assert r.steps == steps
        out[order] = r.T
        tiles[order] = cf.tile_map(case.mesh, case.setup, opts)[0]
    # node renumbering leaves the tiles and every sum order unchanged: bitwise
    assert np.array_equal(tiles["rcm"], tiles["tile"])
    assert np.array_equal(out["rcm"], out["tile"])
    with ThreadPoolExecutor(2) as ex:
        replay = ex.submit(orc.solve, case.mesh, case.setup, steps, tiles["rcm"])
        ref = ex.submit(ref_steps, case.mesh, case.setup, steps) if orc.ref_available() else None
        assert np.array_equal(out["rcm"], replay.result().T), np.abs(out["rcm"] - replay.result().T).max()
        if ref is not None:
            assert rel(out["rcm"], ref.result()) <= RTOL
    assert 299.0 < out["rcm"].min() and out["rcm"].max() < 975.0


def test_cfg3_all_orderings_500_steps():
    """configs[2]: unordered (the given random numbering, tiles = chunks of it), RCM nodes +
    elements by smallest RCM label (the paper's blocks), and the default (first-touch nodes,
    Morton elements): each bitwise equal to the oracle on its tiles, all within 1e-9 of the
    1-block oracle."""
    case = configs.config3()
    steps = case.steps
    assert steps == 500
    orders = {"unordered": dict(node_order="given", elem_order="given"),
              "rcm": dict(node_order="rcm", elem_order="min_node"),
              "default": dict(node_order="tile", elem_order="morton")}
    gpu, tiles = {}, {}
    for k, kw in orders.items():
        opts = cf.SolveOptions(max_steps=steps, **kw)
        gpu[k] = cf.solve(case.mesh, case.setup, opts).T
        tiles[k] = cf.tile_map(case.mesh, case.setup, opts)[0]
    with ThreadPoolExecutor(len(orders) + 1) as ex:
        replays = {k: ex.submit(orc.solve, case.mesh, case.setup, steps, tiles[k]) for k in orders}
        one = ex.submit(orc.solve, case.mesh, case.setup, steps)
        for k in orders:
            rT = replays[k].result().T
            assert np.array_equal(gpu[k], rT), (k, np.abs(gpu[k] - rT).max())
        for k in orders:
            assert rel(gpu[k], one.result().T) <= RTOL, k
    assert not np.array_equal(tiles["unordered"], tiles["default"])


def test_cfg4_three_steps_vs_reference():
    """configs[3] at full size (100,663,296 tets) against the reference solver itself."""
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    case = configs.config4()
    steps = 3
    with ThreadPoolExecutor(1) as ex:
        ref = ex.submit(ref_steps, case.mesh, case.setup, steps)  # ~2 min of reference setup
        gpu = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=steps))
        atomic = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=steps, mode="atomic"))
        r = ref.result()
    assert gpu.steps == steps
    assert rel(gpu.T, r) <= RTOL
    assert rel(atomic.T, r) <= RTOL


def _node_region(tets, region, n):
    reg = np.zeros(n, np.int32)
    reg[tets.reshape(-1)] = np.repeat(region, 4)
    return reg


def test_cfg5_two_steps_vs_oracle_window():
    case = configs.config5()
    steps = 2
    m, s = case.mesh, case.setup
    gpu = cf.solve(m, s, cf.SolveOptions(max_steps=steps))
    assert gpu.steps == steps and np.isfinite(gpu.T).all()
    n = 512
    kz0, kz1, margin = 248, 264, 4
    w = orc.generate_fixture("casting", n, window=[0, n, 0, n, kz0, kz1])
    wm = cf.Mesh(w["nodes"], w["tets"], w["region"], w["facets"], w["facet_tag"], ["outer", "cast_if", "mold_if"],
                 [(1, 2)])
    wreg = _node_region(w["tets"], w["region"], wm.node_count())
    T0 = np.where(wreg == 0, 973.0, 300.0) + orc.counter_uniform(1, w["node_grid"].astype(np.int64), -1.0, 1.0)
    ws = cf.SimulationSetup(materials=s.materials, boundary_conditions=s.boundary_conditions,
                            interface_coeffs=s.interface_coeffs, solver=s.solver, initial_T=T0)
    o = orc.solve(wm, ws, steps)
    assert o.dt == gpu.end_time / steps
    # window node -> full-mesh node by (global grid point, region copy)
    freg = _node_region(m.tets, m.region, m.node_count())
    fkey = m.node_grid.astype(np.int64) * 2 + freg
    order = np.argsort(fkey)
    wkey = w["node_grid"].astype(np.int64) * 2 + wreg
    pos = order[np.searchsorted(fkey, wkey, sorter=order)]
    assert np.array_equal(fkey[pos], wkey)
    P = n + 1
    kz = w["node_grid"] // (P * P)
    inner = (kz >= kz0 + margin) & (kz <= kz1 - margin)
    assert inner.sum() > 1_000_000
    assert rel(gpu.T[pos[inner]], o.T[inner]) <= RTOL
    assert np.array_equal(T0[inner], s.initial_T[pos[inner]])


def test_cfg5_decomposed_matches_single_rank():
    """The 8-rank decomposition of the gate configuration (cfg5, 805 M tets: element ids beyond
    2^29, so 4 x id overflows int32) built by the device pipeline for every rank, all ranks in one
    process on one GPU (in-process transport): 2 steps equal the single-rank run to 1e-9
    (summation order over ranks only)."""
    dc = configs.device_case("cfg5")
    T = {}
    for R in (1, 8):
        with cf.Solver(None, dc.setup, cf.SolveOptions(world_size=R, local_ranks=R), fixture=dc.spec) as s:
            s.step(2)
            T[R] = s.fields(want_H=False)[0]
    assert rel(T[8], T[1]) <= RTOL
