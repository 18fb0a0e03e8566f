"""Physics acceptance checks (SPEC acceptance criteria 2-5; 4-5 against analytic solutions),
through the B200 path: the bitwise parity tests prove the step equals the reference's; these
check that the configured physics (lumped explicit FE, Dirichlet f(t), Lemmon apparent heat
capacity with latent heat) solves the problems SPEC names.

  Fourier bar: unit cube, T0 = sin(pi x), T = 0 on x = 0 and x = 1, adiabatic elsewhere,
               k = rho = c = 1: T = exp(-pi^2 t) sin(pi x); max error <= 1 % of the amplitude.
  Neumann-Stefan: a bar of liquid at the melting point, x = 0 held below it; the solidification
               front s(t) = 2 lambda sqrt(alpha t), lambda e^{lambda^2} erf(lambda) = St/sqrt(pi);
               front within 5 %.
"""
import math

import numpy as np
import pytest

from paper_1005_3158_b200 import castfem as cf

pytestmark = pytest.mark.gpu

KUHN = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def box_mesh(nx, ny, nz, h):
    """Kuhn 6-tet split of an nx x ny x nz grid of cubes of side h; facets on the x = 0 face only
    (tag 0 'cold'); every other face adiabatic (no facet)."""
    P = (nx + 1, ny + 1, nz + 1)
    g = np.stack(np.meshgrid(np.arange(P[0]), np.arange(P[1]), np.arange(P[2]), indexing="ij"), -1)
    nodes = g.transpose(2, 1, 0, 3).reshape(-1, 3).astype(np.float64) * h  # index i + P0 (j + P1 k)
    nid = lambda i, j, k: i + P[0] * (j + P[1] * k)
    tets = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                for a, b, _ in KUHN:
                    v = [[i, j, k], [i, j, k], [i, j, k], [i + 1, j + 1, k + 1]]
                    v[1][a] += 1
                    v[2][a] += 1
                    v[2][b] += 1
                    tets.append([nid(*p) for p in v])
    tets = np.array(tets, np.int32)
    faces = np.concatenate([tets[:, [1, 2, 3]], tets[:, [0, 2, 3]], tets[:, [0, 1, 3]], tets[:, [0, 1, 2]]])
    on = np.all(nodes[faces][:, :, 0] == 0.0, axis=1)
    facets = faces[on]
    return cf.Mesh(nodes, tets, np.zeros(len(tets), np.int32), facets, np.zeros(len(facets), np.int32), ["cold"])


def test_fourier_bar_within_one_percent():
    m = cf.generate_fixture("cube", 16)
    x = m.nodes[m.facets][:, :, 0]
    ends = np.all(x == 0.0, axis=1) | np.all(x == 1.0, axis=1)
    m.facet_tag = np.where(ends, 0, 1).astype(np.int32)
    m.tags = ["ends", "sides"]
    t_end = 0.05
    setup = cf.SimulationSetup(
        materials=[cf.MaterialTable.make(rho=1.0, c=1.0, k=1.0, T0=0.0)],
        boundary_conditions={"ends": cf.BoundaryCondition("fixed", fixed_T=cf.PiecewiseLinear.constant(0.0)),
                             "sides": cf.BoundaryCondition("flux", h=0.0, t_inf=0.0)},
        solver=cf.SolverConfig(dt_safety=0.1, t_end=t_end),
        initial_T=np.sin(np.pi * m.nodes[:, 0]))
    r = cf.solve(m, setup, cf.SolveOptions())
    assert abs(r.end_time - t_end) < 1e-12
    exact = math.exp(-math.pi ** 2 * t_end) * np.sin(np.pi * m.nodes[:, 0])
    err = np.max(np.abs(r.T - exact)) / math.exp(-math.pi ** 2 * t_end)
    assert err <= 0.01, err


def _stefan_lambda(st):
    lo, hi = 1e-6, 3.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if mid * math.exp(mid * mid) * math.erf(mid) < st / math.sqrt(math.pi):
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def test_neumann_stefan_front_within_five_percent():
    h, nx = 0.01, 100
    m = box_mesh(nx, 2, 2, h)
    Tm, Tw, delta, L = 0.0, -1.0, 0.01, 2.0  # Stefan number c (Tm - Tw) / L = 0.5
    mat = cf.MaterialTable.make(rho=1.0, c=1.0, k=1.0, latent_heat=L, solidus=Tm - delta, liquidus=Tm + delta,
                                T0=Tm + delta)
    t_end = 0.185
    setup = cf.SimulationSetup(materials=[mat],
                               boundary_conditions={"cold": cf.BoundaryCondition(
                                   "fixed", fixed_T=cf.PiecewiseLinear.constant(Tw))},
                               solver=cf.SolverConfig(dt_safety=0.1, t_end=t_end))
    r = cf.solve(m, setup, cf.SolveOptions(tile_elems=256))
    axis = (m.nodes[:, 1] == 0.0) & (m.nodes[:, 2] == 0.0)
    xs = m.nodes[axis, 0]
    Ts = r.T[axis][np.argsort(xs)]
    xs = np.sort(xs)
    k = int(np.argmax(Ts >= Tm))  # first node at or above the melting point
    assert 0 < k < len(xs) - 5
    front = xs[k - 1] + (Tm - Ts[k - 1]) / (Ts[k] - Ts[k - 1]) * (xs[k] - xs[k - 1])
    lam = _stefan_lambda(1.0 * (Tm - Tw) / L)
    exact = 2.0 * lam * math.sqrt(r.end_time)
    assert abs(front - exact) / exact <= 0.05, (front, exact)


def test_conservation_1000_steps_and_decomposed_run():
    """SPEC acceptance criteria 2-3 through the B200 path: an adiabatic, constant-property
    10^3-cell cube with a seeded non-uniform T0 conserves sum_i C_i T_i to 1e-10 relative over 1000
    steps (lumped C_i = sum_e rho c V_e / 4), in one rank and split over 3 in-process ranks, and the
    decomposed run equals the single-rank run to 1e-10."""
    from paper_1005_3158_b200 import configs
    c = configs.config1(n=10)
    m = cf.Mesh(c.mesh.nodes, c.mesh.tets, c.mesh.region, np.zeros((0, 3)), np.zeros(0), [])
    rng = np.random.default_rng(7)
    T0 = 600.0 + 300.0 * rng.random(m.node_count())
    s = cf.SimulationSetup(materials=c.setup.materials, solver=c.setup.solver, initial_T=T0)
    tets, _ = cf.finalize_mesh(m)
    p = m.nodes[tets]
    V = np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0])) / 6
    Cn = np.zeros(m.node_count())
    np.add.at(Cn, tets.reshape(-1), np.repeat(2700.0 * 900.0 * V / 4, 4))
    one = cf.solve(m, s, cf.SolveOptions(max_steps=1000, tile_elems=256))
    dd = cf.solve(m, s, cf.SolveOptions(max_steps=1000, tile_elems=256, world_size=3, local_ranks=3))
    assert one.steps == dd.steps == 1000
    for r in (one, dd):
        assert abs(np.sum(Cn * (r.T - T0))) <= 1e-10 * np.sum(Cn * T0)
        assert np.ptp(r.T) < np.ptp(T0)  # diffusion only smooths
    assert float(np.max(np.abs(dd.T - one.T) / np.abs(one.T))) <= 1e-10


def test_permuted_mesh_gives_the_permuted_solution():
    """solving on permute_mesh(m, p) equals the permuted solution of m to 1e-12
    (node renumbering only relabels the unknowns) -- with the RCM permutation from the device pass and
    with a random one, on a jittered two-material casting."""
    from paper_1005_3158_b200 import configs
    c = configs.casting(10, jitter=0.15, seed=4, dt_safety=0.14)
    m, s = c.mesh, c.setup
    base = cf.solve(m, s, cf.SolveOptions(max_steps=60, tile_elems=256))
    rng = np.random.default_rng(11)
    for p in (cf.rcm_permutation_device(m), rng.permutation(m.node_count()).astype(np.int32)):
        mp = cf.permute_mesh(m, p)
        T0p = np.empty_like(s.initial_T)
        T0p[p] = s.initial_T
        sp = cf.SimulationSetup(materials=s.materials, boundary_conditions=s.boundary_conditions,
                                interface_coeffs=s.interface_coeffs, solver=s.solver, initial_T=T0p)
        r = cf.solve(mp, sp, cf.SolveOptions(max_steps=60, tile_elems=256))
        assert float(np.max(np.abs(r.T[p] - base.T) / np.abs(base.T))) <= 1e-12
        assert r.end_time == base.end_time
