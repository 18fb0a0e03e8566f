"""Rank-local setup at scale: W processes on ONE GPU (host-staged exchange over gloo: NCCL refuses
two ranks on one device), each generating the cfg4 mesh on the device and building only its RCB
part; per-process setup time and peak host RSS, whole-mesh T after K steps compared with the
single-process run (<= 1e-9: the summation order over ranks differs).
    python scripts/multiproc_fixture.py 2 10 [cfg]"""
import json
import multiprocessing as mp
import os
import resource
import socket
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, cfg, steps, out):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_1005_3158_b200 import castfem as cf
    from paper_1005_3158_b200 import configs
    dc = configs.device_case(cfg)
    comm = cf.HostComm(world, rank, 0) if world > 1 else None
    t0 = time.time()
    opts = cf.SolveOptions(world_size=world, rank=rank, local_ranks=1, comm=comm)
    with cf.Solver(None, dc.setup, opts, fixture=dc.spec) as s:
        setup = time.time() - t0
        rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
        st = s.stats()
        s.step(steps)
        T = np.full(st.n_nodes_global, np.nan)
        s.fields(want_H=False, out=(T, None))
        st2 = s.stats()
    if comm:
        comm.close()
    np.savez(out, T=T, info=np.array([setup, rss, st.n_elems_local, st.n_nodes_local, st.device_bytes,
                                      st2.loop_seconds]))
    dist.destroy_process_group()


def run(world, cfg, steps, tag):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    outs = [f"/tmp/mpf_{tag}_{r}.npz" for r in range(world)]
    ps = [ctx.Process(target=worker, args=(r, world, port, cfg, steps, outs[r])) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join()
        if p.exitcode:
            raise SystemExit(f"rank failed: {p.exitcode}")
    T = None
    info = []
    for o in outs:
        d = np.load(o)
        T = d["T"] if T is None else np.where(np.isnan(T), d["T"], T)
        info.append(d["info"].tolist())
    return T, info


if __name__ == "__main__":
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg4"
    T1, i1 = run(1, cfg, steps, "one")
    TW, iW = run(W, cfg, steps, "many")
    rel = float(np.nanmax(np.abs(TW - T1) / np.abs(T1)))
    keys = ["setup_s", "host_peak_rss_gb", "elems_local", "nodes_local", "device_bytes", "loop_s"]
    print(json.dumps({"config": cfg, "world": W, "steps": steps, "transport": "host-staged (gloo), all ranks on cuda:0",
                      "single_process": dict(zip(keys, i1[0])),
                      "ranks": [dict(zip(keys, x)) for x in iW], "all_nodes_covered": bool(not np.isnan(TW).any()),
                      "max_rel_vs_single_process": rel, "pass": rel <= 1e-9}))
