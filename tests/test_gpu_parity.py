"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Tolerance (north_star): nodal T within 1e-9 relative of the oracle in atomic
mode; deterministic mode is bitwise equal to the oracle replaying the same
tiles as BlockPlan blocks (the reference's blocked semantics,
blocked.hpp:217-307, 502-515) and bitwise reproducible run to run.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1005_3158_b200 import castfem as cf
from paper_1005_3158_b200 import configs

pytestmark = pytest.mark.gpu
RTOL = 1e-9


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


def run_pair(case, steps, tile_elems=512, **kw):
    det_opts = cf.SolveOptions(max_steps=steps, mode="deterministic", tile_elems=tile_elems, **kw)
    det = cf.solve(case.mesh, case.setup, det_opts)
    tiles, _ = cf.tile_map(case.mesh, case.setup, det_opts)
    ref = orc.solve(case.mesh, case.setup, steps, blocks=tiles)
    return det, ref


GEOMS = ["coords", "stored"]  # gradients recomputed from slot coordinates | stored ElementGeom


@pytest.mark.parametrize("geometry", GEOMS)
@pytest.mark.parametrize("n", [8, 16])
def test_cfg1_cube_deterministic_bitwise(n, geometry):
    case = configs.config1(n=n)
    det, ref = run_pair(case, 30, geometry=geometry)
    assert np.array_equal(det.T, ref.T), np.abs(det.T - ref.T).max()
    assert np.array_equal(det.H, ref.H)
    assert det.steps == ref.steps == 30
    assert det.end_time == ref.time


@pytest.mark.parametrize("geometry", GEOMS)
@pytest.mark.parametrize("n,jitter,perm", [(12, 0.0, 0), (14, 0.2, 5)])
def test_casting_deterministic_bitwise(n, jitter, perm, geometry):
    case = configs.casting(n, jitter=jitter, seed=3, perm_seed=perm, dt_safety=0.14)
    det, ref = run_pair(case, 40, geometry=geometry)
    assert np.array_equal(det.T, ref.T), np.abs(det.T - ref.T).max()


@pytest.mark.parametrize("order,geometry", [("morton", "coords"), ("min_node", "coords"), ("given", "coords"),
                                            ("morton", "stored")])
def test_casting_atomic_within_tolerance(order, geometry):
    case = configs.casting(14, jitter=0.2, seed=3, perm_seed=9, dt_safety=0.14)
    at = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=40, mode="atomic", elem_order=order,
                                                         geometry=geometry))
    ref = orc.solve(case.mesh, case.setup, 40)
    assert rel(at.T, ref.T) <= RTOL


def test_deterministic_repeat_bitwise():
    case = configs.casting(16, dt_safety=0.14)
    a = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=25, mode="deterministic"))
    b = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=25, mode="deterministic"))
    assert np.array_equal(a.T, b.T)


@pytest.mark.parametrize("env", [{"CF_TILE_PERSIST": "0"}, {"CF_TILE_DYNAMIC": "0"}, {"CF_BANK_ITERS": "4"},
                                 {"CF_BANK_PASSES": "3"}, {"CF_SLOT_ORDER": "count"}, {"CF_SLOT_BANKS": "0"},
                                 {"CF_TILE_PERSIST": "0", "CF_BANK_ITERS": "0"}, {"CF_SLOT_GATHER": "1"},
                                 {"CF_L2_NEXT": "0"}, {"CF_TILE_STAGES": "2"}, {"CF_TILE_ORDER": "morton"},
                                 {"CF_HOST_SETUP": "1"}])
def test_schedule_and_element_positions_leave_results_bitwise(env, monkeypatch):
    """Persistent (dynamically or statically scheduled) vs one-CTA-per-tile grids and the
    bank-aware element positions inside a tile (greedy colouring, optional local search) only
    move work and shared-memory addresses: the reduction order is the CSR's, so T is bitwise that
    of the default plan and the oracle. 40^3 cells: ~1000 tiles, several per persistent CTA."""
    case = configs.casting(40, jitter=0.2, seed=3, perm_seed=5, dt_safety=0.14)
    opts = cf.SolveOptions(max_steps=30, mode="deterministic", tile_elems=384)
    base = cf.solve(case.mesh, case.setup, opts)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    alt = cf.solve(case.mesh, case.setup, opts)
    assert np.array_equal(base.T, alt.T), np.abs(base.T - alt.T).max()
    tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
    ref = orc.solve(case.mesh, case.setup, 30, blocks=tiles)
    assert np.array_equal(alt.T, ref.T)


def test_reference_blocks_replayed():
    """GPU tiles = the reference's own partition_graph blocks -> bitwise equal to the reference."""
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    case = configs.casting(10, dt_safety=0.14)
    ref, bm = orc.ref_solve(case.mesh, case.setup, 30, blocks=8)
    det = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=30, mode="deterministic", blocks=bm))
    assert np.array_equal(det.T, ref.T)


# ---------------------------------------------------------------- domain decomposition
@pytest.mark.parametrize("ranks", [2, 4])
@pytest.mark.parametrize("mode", ["deterministic", "atomic"])
def test_multirank_inprocess_vs_oracle(ranks, mode):
    """RCB decomposition over `ranks` in-process ranks on one GPU (exchange of
    shared-node partials + external-node T by device copies): deterministic
    mode is bitwise equal to the oracle replaying the same parts and tiles
    (per node: ascending-rank sum of each rank's ascending-tile partial)."""
    case = configs.casting(12, jitter=0.15, seed=2, dt_safety=0.14)
    parts = cf.partition_rcb(case.mesh, ranks)
    opts = cf.SolveOptions(max_steps=30, mode=mode, tile_elems=256, world_size=ranks, local_ranks=ranks)
    gpu = cf.solve(case.mesh, case.setup, opts)
    tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
    ref = orc.solve(case.mesh, case.setup, 30, blocks=tiles, parts=parts)
    if mode == "deterministic":
        assert np.array_equal(gpu.T, ref.T), np.abs(gpu.T - ref.T).max()
    assert rel(gpu.T, ref.T) <= RTOL
    single = orc.solve(case.mesh, case.setup, 30)
    assert rel(gpu.T, single.T) <= RTOL


def test_multirank_fused_border_launch(monkeypatch):
    """CF_BORDER_FUSED=1: one tile launch per rank, border tiles first; the kernel raises a flag
    when its last border tile has flushed and the exchange stream waits on the flag's value
    before packing. Same tiles, same reduction order: bitwise equal to the default two-launch
    schedule and to the oracle with the same parts."""
    case = configs.casting(16, jitter=0.15, seed=2, dt_safety=0.14)
    opts = cf.SolveOptions(max_steps=30, mode="deterministic", tile_elems=192, world_size=3, local_ranks=3)
    base = cf.solve(case.mesh, case.setup, opts)
    monkeypatch.setenv("CF_BORDER_FUSED", "1")
    fused = cf.solve(case.mesh, case.setup, opts)
    assert np.array_equal(base.T, fused.T)
    tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
    ref = orc.solve(case.mesh, case.setup, 30, blocks=tiles, parts=cf.partition_rcb(case.mesh, 3))
    assert np.array_equal(fused.T, ref.T)


def test_multirank_interface_split_across_ranks():
    """A partition cutting through the cast/mould interface: sister elements on
    other ranks supply the lagged ambient through ghost nodes."""
    case = configs.casting(10, dt_safety=0.14)
    E = case.mesh.element_count()
    parts = (np.arange(E) % 3).astype(np.int32)  # scattered parts: every interface pair crosses ranks
    opts = cf.SolveOptions(max_steps=20, mode="deterministic", tile_elems=128, world_size=3, local_ranks=3,
                           part_of_element=parts)
    gpu = cf.solve(case.mesh, case.setup, opts)
    tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
    ref = orc.solve(case.mesh, case.setup, 20, blocks=tiles, parts=parts)
    assert np.array_equal(gpu.T, ref.T)


# ---------------------------------------------------------------- solver semantics
def test_t_end_mode_and_series():
    """solve_serial's t_end loop (blocked.hpp:674-677): dt clipped to the
    remaining time, output_every series of (t, Tmin, Tmax)."""
    case = configs.casting(10, dt_safety=0.14)
    case.setup.solver.output_every = 7
    dt = orc.solve(case.mesh, case.setup, 1).dt
    case.setup.solver.t_end = 23.5 * dt
    gpu = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=0))
    ref = orc.solve(case.mesh, case.setup, 0)
    assert gpu.steps == ref.steps == 24
    assert gpu.end_time == ref.time
    assert rel(gpu.T, ref.T) <= RTOL
    assert len(gpu.series) == len(ref.series) == 3
    for s, r in zip(gpu.series, ref.series):
        assert s.time == r[0] and abs(s.t_min - r[1]) <= 1e-9 * abs(r[1]) and abs(s.t_max - r[2]) <= 1e-9 * r[2]


def _dirichlet_tdep_case():
    m = cf.generate_fixture("cube", 8)
    # split the outer tag: x = 0 face fixed, the rest convective
    x0 = np.all(m.nodes[m.facets][:, :, 0] == 0.0, axis=1)
    m.facet_tag = np.where(x0, 1, 0).astype(np.int32)
    m.tags = ["outer", "hot"]
    mat = cf.MaterialTable.make(rho=7800.0, c=[(300.0, 450.0), (900.0, 700.0)], k=[(300.0, 45.0), (900.0, 30.0)],
                                latent_heat=2.0e5, solidus=700.0, liquidus=760.0, T0=650.0)
    setup = cf.SimulationSetup(
        materials=[mat],
        boundary_conditions={"outer": cf.BoundaryCondition("flux", h=50.0, t_inf=300.0),
                             "hot": cf.BoundaryCondition("fixed", fixed_T=cf.PiecewiseLinear([0.0, 50.0], [650.0, 950.0]))},
        solver=cf.SolverConfig(dt_safety=0.1))
    return m, setup


@pytest.mark.parametrize("geometry", GEOMS)
def test_dirichlet_and_temperature_dependent_tables(geometry):
    """Fixed-temperature BC f(t) (lowest tag wins, blocked.hpp:250-263),
    piecewise-linear c(T), k(T) (dynamic dt, :477-480) and clamp accounting."""
    m, setup = _dirichlet_tdep_case()
    opts = cf.SolveOptions(max_steps=60, tile_elems=128, geometry=geometry)
    gpu = cf.solve(m, setup, opts)
    tiles, _ = cf.tile_map(m, setup, opts)
    ref = orc.solve(m, setup, 60, blocks=tiles)
    assert gpu.steps == 60 and gpu.end_time == ref.time
    assert np.array_equal(gpu.T, ref.T), np.abs(gpu.T - ref.T).max()
    assert rel(gpu.T, orc.solve(m, setup, 60).T) <= RTOL
    assert gpu.clamp_steps == ref.clamp_steps and ref.clamp_steps > 0


@pytest.mark.parametrize("ranks", [2, 3])
def test_multirank_dynamic_dt(ranks):
    """Dynamic dt on a decomposed mesh: every rank steps with the min of the stable bound over
    the whole mesh (blocked.hpp:477-480) -- min-combined across ranks each step (in-process
    here; ncclAllReduce(min) across processes). Bitwise equal to the oracle with the same parts."""
    m, setup = _dirichlet_tdep_case()
    parts = cf.partition_rcb(m, ranks)
    opts = cf.SolveOptions(max_steps=60, tile_elems=128, world_size=ranks, local_ranks=ranks)
    gpu = cf.solve(m, setup, opts)
    tiles, _ = cf.tile_map(m, setup, opts)
    ref = orc.solve(m, setup, 60, blocks=tiles, parts=parts)
    assert gpu.steps == 60 and gpu.end_time == ref.time
    assert np.array_equal(gpu.T, ref.T), np.abs(gpu.T - ref.T).max()
    assert gpu.clamp_steps == ref.clamp_steps


@pytest.mark.parametrize("geometry", GEOMS)
def test_lambda_max_matches_oracle(geometry):
    case = configs.casting(10, dt_safety=0.14)
    with cf.Solver(case.mesh, case.setup, cf.SolveOptions(geometry=geometry)) as s:
        lam, e13 = s.estimate_lambda_max(300)
    lo, e13o = orc.lambda_max(case.mesh, case.setup, 300)
    assert abs(lam - lo) <= 1e-6 * lo
    assert e13 == e13o


def test_cpp_drop_in_example():
    """A reference user's C++ program: castfem::solve_serial vs castfem_b200::solve_gpu on the
    reference's own Mesh / SimulationSetup objects (initial_override, Dirichlet f(t), c(T) table,
    series, clamp accounting, reference exception types through the shim)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(orc.__file__), "_ref", "drop_in_example")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/drop_in_example not built (needs the reference headers at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout


# ---------------------------------------------------------------- BASELINE sizes
@pytest.mark.slow
def test_cfg1_full_size_vs_oracle():
    """BASELINE configs[0]: 32^3 cube, 100 steps, dt = 0.9 x 2/lambda_max."""
    case = configs.config1(32)
    det, ref = run_pair(case, case.steps, tile_elems=384)
    assert np.array_equal(det.T, ref.T)
    assert det.steps == 100
    one = orc.solve(case.mesh, case.setup, case.steps)
    assert rel(det.T, one.T) <= RTOL


@pytest.mark.slow
def test_cfg2_full_size_vs_reference_truncated():
    """BASELINE configs[1] (12.6 M tets): 10 steps against the reference solver itself."""
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    case = configs.config2()
    gpu = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=10))
    rb = orc.RefBench(case.mesh, case.setup)
    rb.steps(10)
    ref = rb.T()
    rb.close()
    assert rel(gpu.T, ref) <= RTOL


@pytest.mark.slow
def test_cfg2_bit_reproducible_run_to_run():
    case = configs.config2()
    with cf.Solver(case.mesh, case.setup) as s:
        s.step(50)
        a, _ = s.fields(False)
        s.set_temperature(case.setup.initial_T)
        s.step(50)
        b, _ = s.fields(False)
    assert np.array_equal(a, b)
    assert np.isfinite(a).all() and 299.0 < a.min() and a.max() < 975.0


def test_graph_replay_bitwise():
    """CUDA-graph stepping (captured 6-step graphs, replayed; remainder steps eager) is bitwise
    equal to stream stepping, including a step count that is not a multiple of the graph."""
    case = configs.casting(12, dt_safety=0.14)
    plain = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=29))
    graph = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=29, graph_steps=6))
    assert np.array_equal(plain.T, graph.T)
    assert plain.end_time == graph.end_time and plain.steps == graph.steps == 29


@pytest.mark.slow
def test_cfg4_full_size_properties():
    """BASELINE configs[3] (256^3 cells, 100,663,296 tets) on one GPU, through size-independent
    properties (the oracle is too slow at this size): the sum-order-sensitive variants -- fp64 RED
    accumulation, the coordinates tile layout (its own tiling), two ranks in one process (RCB halves
    plus the exchange combine) -- agree with the deterministic single-rank run within the north_star
    1e-9, and the deterministic run is bit-reproducible."""
    case = configs.config4()
    steps = 20
    base = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=steps))
    assert base.steps == steps and np.isfinite(base.T).all()
    assert 299.0 < base.T.min() and base.T.max() < 975.0
    again = cf.solve(case.mesh, case.setup, cf.SolveOptions(max_steps=steps))
    assert np.array_equal(base.T, again.T)
    del again
    variants = [cf.SolveOptions(max_steps=steps, mode="atomic"),
                cf.SolveOptions(max_steps=steps, geometry="coords"),
                cf.SolveOptions(max_steps=steps, world_size=2, local_ranks=2)]
    for opts in variants:
        other = cf.solve(case.mesh, case.setup, opts)
        assert other.end_time == base.end_time
        assert rel(other.T, base.T) <= RTOL, opts


def test_autotune_tiles():
    """autotune_block_count recast: every candidate is planned and timed (best of 2), an
    infeasible one (2048 stored tets exceed shared memory) times +inf, the fastest is chosen,
    and stepping with the chosen tile size stays bitwise equal to the oracle on its tiles."""
    case = configs.casting(14, dt_safety=0.14)
    rep = cf.autotune_tiles(case.mesh, case.setup, candidates=[192, 384, 2048], trial_steps=5,
                            projected_total_steps=1000)
    assert rep.candidates == [192, 384, 2048]
    assert np.isfinite(rep.seconds[0]) and np.isfinite(rep.seconds[1]) and rep.seconds[2] == float("inf")
    assert rep.chosen == cf.choose_tile_elems(rep.candidates, rep.seconds) and rep.chosen in (192, 384)
    assert 0.0 < rep.overhead_fraction < 1.0
    det, ref = run_pair(case, 20, tile_elems=rep.chosen)
    assert np.array_equal(det.T, ref.T)


def test_fields_into_caller_buffers():
    """Solver.fields(out=...) fills caller-owned (e.g. pinned) arrays with the same values."""
    case = configs.casting(10, dt_safety=0.14)
    with cf.Solver(case.mesh, case.setup) as s:
        s.step(7)
        T, H = s.fields()
        To, Ho = np.empty_like(T), np.empty_like(H)
        T2, H2 = s.fields(out=(To, Ho))
        assert T2 is To and H2 is Ho
        assert np.array_equal(To, T) and np.array_equal(Ho, H)
        with pytest.raises(ValueError):
            s.fields(out=(np.empty(3), None))


@pytest.mark.parametrize("n", [24, 40])
def test_uniform_t0_degeneracy_matches_reference(n):
    """BASELINE's literal uniform casting T0 (no noise): the hot interior varies by round-off
    only, so the Lemmon degeneracy test (fem.hpp:36-44) decides on near-zero gradients, where
    the stored layout's 1/|g1| bound cannot and the exact max_edge is fetched from the blob's
    uncopied tail. Bitwise equal to the oracle replaying the same tiles (cfg2 itself throws
    "zero lumped capacitance" at step 30, node 802288, in the reference and here alike)."""
    case = configs.casting(n, noise=0.0, dt_safety=0.138)
    for geometry in ("stored", "coords"):
        det, ref = run_pair(case, 80, tile_elems=384, geometry=geometry)
        assert np.array_equal(det.T, ref.T), np.abs(det.T - ref.T).max()


def test_stepping_paths_share_the_dynamic_schedule():
    """The persistent tile kernel's scheduling counter is reset by every step's advance kernel,
    whichever API drives the steps: step(), time_phases() and fields() interleaved on ~1000 tiles
    (several per CTA) stay bitwise equal to the oracle replaying the same tiles."""
    case = configs.casting(40, jitter=0.2, seed=21, perm_seed=7, dt_safety=0.17)
    opts = cf.SolveOptions(mode="deterministic")
    with cf.Solver(case.mesh, case.setup, opts) as sv:
        sv.step(5)
        T5, _ = sv.fields(False)
        sv.time_phases(10)
        sv.step(20)
        T35, _ = sv.fields(False)
        assert sv.stats().step_index == 35
    tiles, nt = cf.tile_map(case.mesh, case.setup, opts)
    assert nt > 600  # more tiles than resident CTAs: the dynamic scheduler is active
    assert np.array_equal(T5, orc.solve(case.mesh, case.setup, 5, blocks=tiles).T)
    assert np.array_equal(T35, orc.solve(case.mesh, case.setup, 35, blocks=tiles).T)


def test_multirank_graph_partition_vs_oracle():
    """A decomposition by the reference's partitioner (greedy graph growing over the dual graph
    glued by virtual interface elements, partition="graph") instead of RCB: 3 in-process ranks,
    bitwise equal to the oracle replaying the same parts and tiles."""
    case = configs.casting(12, jitter=0.2, seed=4, perm_seed=2, dt_safety=0.14)
    parts = cf.partition_elements(case.mesh, 3)
    opts = cf.SolveOptions(max_steps=25, tile_elems=192, world_size=3, local_ranks=3, partition="graph")
    gpu = cf.solve(case.mesh, case.setup, opts)
    tiles, _ = cf.tile_map(case.mesh, case.setup, opts)
    assert np.array_equal(np.unique(parts), [0, 1, 2])
    ref = orc.solve(case.mesh, case.setup, 25, blocks=tiles, parts=parts)
    assert np.array_equal(gpu.T, ref.T), np.abs(gpu.T - ref.T).max()
