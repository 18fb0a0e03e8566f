"""The multi-rank exchange protocol on CPU with torch.distributed (gloo).

Each process is one rank of an RCB decomposition. It takes its neighbour
lists from the PRODUCT's plan builder (cf_exchange_plan: the same lists the
GPU pack/update kernels use), assembles its own elements with the oracle,
swaps [c(shared) | r(shared) | T(ext_to)] with every neighbour (SPEC
exchange_and_merge S:450-458; payload 2*shared + external), sums shared
nodes in ascending rank order, updates, and refreshes ghost T for the lagged
ambient. The result must equal the single-process oracle with the same parts
bit for bit, and the single-domain oracle to 1e-15.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_1005_3158_b200 import configs
    return configs.casting(9, jitter=0.1, seed=6, dt_safety=0.14)


def _worker(rank, world, port, steps, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_1005_3158_b200 import castfem as cf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    case = _case()
    m, s = case.mesh, case.setup
    parts = cf.partition_rcb(m, world)
    plan = cf.exchange_plan(m, s, world, rank, parts)
    mask = (parts == rank).astype(np.int8)
    mine = np.unique(m.tets[parts == rank].reshape(-1))
    on = np.zeros((world, m.node_count()), bool)
    for p in range(world):
        on[p, np.unique(m.tets[parts == p].reshape(-1))] = True
    dt = orc.solve(m, s, 1).dt
    T = s.initial_T.copy() if s.initial_T is not None else np.array(
        [s.materials[r].initial_temperature for r in np.bincount(m.tets.reshape(-1), minlength=m.node_count()) * 0])
    T_old = T.copy()
    time = 0.0
    for _ in range(steps):
        c, r = orc.assemble_part(m, s, mask, T, T_old, time)
        reqs, recv = [], {}
        for x in plan:  # one message per neighbour, both directions
            send = np.concatenate([c[x["shared"]], r[x["shared"]], T[x["ext_to"]]])
            rb = torch.empty(2 * len(x["shared"]) + len(x["ext_from"]), dtype=torch.float64)
            reqs.append(dist.isend(torch.from_numpy(send), x["rank"]))
            reqs.append(dist.irecv(rb, x["rank"]))
            recv[x["rank"]] = rb
        for q in reqs:
            q.wait()
        ct, rt = c.copy(), r.copy()
        shared_nodes = np.unique(np.concatenate([x["shared"] for x in plan])) if plan else np.zeros(0, int)
        for n in shared_nodes:  # ascending-rank sum on every replica
            acc_c, acc_r = 0.0, 0.0
            for p in range(world):
                if not on[p, n]:
                    continue
                if p == rank:
                    acc_c += c[n]
                    acc_r += r[n]
                else:
                    x = next(y for y in plan if y["rank"] == p)
                    j = int(np.searchsorted(x["shared"], n))
                    rb = recv[p].numpy()
                    acc_c += rb[j]
                    acc_r += rb[len(x["shared"]) + j]
            ct[n], rt[n] = acc_c, acc_r
        T_old = T.copy()  # pre-update T: next step's ambient source
        for x in plan:
            rb = recv[x["rank"]].numpy()
            T_old[x["ext_from"]] = rb[2 * len(x["shared"]):]
        T = T.copy()
        T[mine] = T[mine] + dt * rt[mine] / ct[mine]
        time += dt
    out[rank] = (mine, T[mine])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_matches_oracle(world):
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    from paper_1005_3158_b200 import castfem as cf
    steps = 6
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, steps, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    case = _case()
    parts = cf.partition_rcb(case.mesh, world)
    ref = orc.solve(case.mesh, case.setup, steps, blocks=parts, parts=parts)
    single = orc.solve(case.mesh, case.setup, steps)
    for r in range(world):
        nodes, T = out[r]
        assert np.array_equal(T, ref.T[nodes]), np.abs(T - ref.T[nodes]).max()
        assert np.max(np.abs(T - single.T[nodes]) / single.T[nodes]) < 1e-14


def _host_comm_worker(rank, world, port, out):
    """The product's host-staged transport callbacks (castfem.HostComm, the functions the library
    calls from cf_step) driven directly with payloads of the exchange plan's shape."""
    sys.path.insert(0, ROOT)
    import ctypes as C

    import torch.distributed as dist

    from paper_1005_3158_b200 import castfem as cf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = cf.HostComm(world, rank, 0)
    sendrecv, allreduce = comm._cb
    peers = [q for q in range(world) if q != rank]
    n = len(peers)
    send = [np.arange(5 + q, dtype=np.float64) + 100 * rank + 10 * q for q in peers]   # rank -> q
    recv = [np.full(5 + rank, np.nan) for q in peers]                                    # q -> rank
    dp = C.POINTER(C.c_double)
    rc = sendrecv(None, n, (C.c_int32 * n)(*peers), (dp * n)(*[a.ctypes.data_as(dp) for a in send]),
                  (C.c_int64 * n)(*[a.size for a in send]), (dp * n)(*[a.ctypes.data_as(dp) for a in recv]),
                  (C.c_int64 * n)(*[a.size for a in recv]))
    vals = np.array([float(rank + 1), -float(rank)])
    rc2 = allreduce(None, vals[:1].ctypes.data_as(dp), 1, 0)  # min
    rc3 = allreduce(None, vals[1:].ctypes.data_as(dp), 1, 1)  # max
    out[rank] = (rc, rc2, rc3, [r.tolist() for r in recv], vals.tolist())
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_comm_callbacks(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_host_comm_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    for r in range(world):
        rc, rc2, rc3, recv, vals = out[r]
        assert (rc, rc2, rc3) == (0, 0, 0)
        peers = [q for q in range(world) if q != r]
        for q, got in zip(peers, recv):
            assert got == (np.arange(5 + r, dtype=np.float64) + 100 * q + 10 * r).tolist()
        assert vals == [1.0, 0.0]
