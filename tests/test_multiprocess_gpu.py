"""Multi-process decomposition through the product path: one process per rank, every rank on
cuda:0, the exchange_and_merge payload moved by the host-staged transport
(cf_comm_create_host over a gloo process group; NCCL refuses two ranks on one device) or by the
peer-memory transport (cf_comm_create_peer: the pack kernel stores into the neighbours'
IPC-exported windows and raises step flags the neighbours' streams wait on).

Each process builds only its own rank's plan (local_ranks = 1), steps, and writes the nodes it
owns; the merged field must be bitwise equal to the oracle replaying the same parts and tiles
(per node: ascending-rank sum of each rank's ascending-tile partial), replicas of shared nodes
bitwise identical, and the whole-mesh statistics (clamp steps, series T_min / T_max, dynamic dt)
equal on every rank. No kernel waits on another process's kernel: the ranks meet on the host
(host-staged) or their streams wait on flag values (peer memory: cuStreamWaitValue32 holds the
stream, not an SM, so the processes time-slicing one GPU cannot block each other).
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(kind):
    from paper_1005_3158_b200 import configs
    if kind == "casting":
        case = configs.casting(12, jitter=0.15, seed=2, dt_safety=0.14, steps=30)
        return case.mesh, case.setup
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_parity import _dirichlet_tdep_case
    return _dirichlet_tdep_case()


def _worker(rank, world, port, kind, steps, mode, out, transport="host"):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_1005_3158_b200 import castfem as cf
        mesh, setup = _case(kind)
        setup.solver.output_every = 10
        comm = (cf.PeerComm if transport == "peer" else cf.HostComm)(world, rank, 0)
        opts = cf.SolveOptions(max_steps=steps, mode=mode, tile_elems=128, world_size=world, rank=rank,
                               local_ranks=1, comm=comm)
        with cf.Solver(mesh, setup, opts) as s:
            series = s.solve(steps)
            T = np.full(mesh.node_count(), np.nan)
            s.fields(want_H=False, out=(T, None))
            st = s.stats()
            stats = np.array([st.time, st.step_index, st.clamp_steps, st.n_elems_local, st.n_shared_nodes])
        comm.close()
        ser = np.array([[x.time, x.t_min, x.t_max] for x in series]).reshape(-1, 3)
        np.savez(out, T=T, stats=stats, series=ser)
    finally:
        dist.destroy_process_group()


def _run(kind, world, steps, mode, tmp_path, transport="host"):
    port = _free_port()
    ctx = mp.get_context("spawn")
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(world)]
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, steps, mode, outs[r], transport)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for p in procs:
        if p.is_alive():
            p.kill()
        assert p.exitcode == 0, f"rank process exited with {p.exitcode}"
    return [np.load(o) for o in outs]


def _merge(res):
    T = np.full(res[0]["T"].shape, np.nan)
    for r in res:
        v = r["T"]
        have = ~np.isnan(v)
        both = have & ~np.isnan(T)
        assert np.array_equal(T[both], v[both]), "replicas of a shared node differ"
        T[have] = v[have]
    assert not np.isnan(T).any(), "some node is owned by no rank"
    return T


@pytest.mark.parametrize("transport", ["host", "peer"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["deterministic", "atomic"])
def test_host_transport_processes_vs_oracle(world, mode, transport, tmp_path):
    from oracle import oracle as orc
    from paper_1005_3158_b200 import castfem as cf
    steps = 30
    res = _run("casting", world, steps, mode, tmp_path, transport)
    T = _merge(res)
    mesh, setup = _case("casting")
    setup.solver.output_every = 10
    parts = cf.partition_rcb(mesh, world)
    opts = cf.SolveOptions(tile_elems=128, world_size=world, local_ranks=world, mode=mode)
    tiles, _ = cf.tile_map(mesh, setup, opts)
    ref = orc.solve(mesh, setup, steps, blocks=tiles, parts=parts)
    if mode == "deterministic":
        assert np.array_equal(T, ref.T), np.abs(T - ref.T).max()
    assert float(np.max(np.abs(T - ref.T) / np.abs(ref.T))) <= 1e-9
    # each process stepped only its own part; the statistics cover the whole mesh on every rank
    assert sum(int(r["stats"][3]) for r in res) == mesh.element_count()
    for r in res:
        assert r["stats"][0] == ref.time and int(r["stats"][1]) == steps
        assert r["series"].shape == (3, 3)
        assert np.array_equal(r["series"], res[0]["series"])
    assert np.array_equal(res[0]["series"][:, 0], ref.series[:, 0])
    assert np.allclose(res[0]["series"][:, 1:], ref.series[:, 1:], rtol=1e-9, atol=0)


@pytest.mark.parametrize("transport", ["host", "peer"])
def test_host_transport_dynamic_dt_and_clamps(transport, tmp_path):
    """Temperature-dependent tables: the per-step stable bound is min-reduced over the processes
    (blocked.hpp:477-480 is a min over the whole mesh) and a step counts as clamped when any
    rank's node clamps (blocked.hpp:526-534) -- identical on every rank, equal to the oracle."""
    from oracle import oracle as orc
    from paper_1005_3158_b200 import castfem as cf
    steps, world = 60, 2
    res = _run("tdep", world, steps, "deterministic", tmp_path, transport)
    T = _merge(res)
    mesh, setup = _case("tdep")
    parts = cf.partition_rcb(mesh, world)
    opts = cf.SolveOptions(tile_elems=128, world_size=world, local_ranks=world)
    tiles, _ = cf.tile_map(mesh, setup, opts)
    ref = orc.solve(mesh, setup, steps, blocks=tiles, parts=parts)
    assert np.array_equal(T, ref.T), np.abs(T - ref.T).max()
    assert ref.clamp_steps > 0
    for r in res:
        assert r["stats"][0] == ref.time
        assert int(r["stats"][2]) == ref.clamp_steps
