#!/usr/bin/env python3
"""Benchmark of the B200 castfem explicit step (one JSON line on rank 0).

A "step" is one explicit time step (blocked_step, blocked.hpp:542-550) over
the whole synthetic mesh: element/facet assembly + merge + update.

Workload (seeded synthetic meshes, no external data): BASELINE
configs[4] = cfg5, the 512^3-cell casting (805,306,368 tets, 135.6 M nodes), the
largest configuration and the one the 1/2/4/8-GPU metric is quoted on; it fits one
B200 (~105 GB). N = 1 steps it on one GPU; N > 1 is strong scaling of the SAME mesh:
recursive coordinate bisection into N parts, one rank per GPU, one NCCL exchange of
interface-node partials per step. --config cfg1..cfg4 selects another config.

value  = element-updates/s over the K timed steps, inputs resident in HBM
         (device time by CUDA events on the plan's stream; max over ranks).
e2e    = the same metric through the public API with pinned host buffers:
         set_temperature(host T0) -> step(K) -> fields(host T, H).
--impl reference times the reference solver itself (oracle/_ref/ref_bench: the
         unmodified castfem headers + the oracle's workload generator, its own process;
         this process never loads the product library) on the host: rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import resource
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# host setup (mesh generation, validation, tiling) is OpenMP-parallel; torchrun
# pins OMP_NUM_THREADS=1, so give each rank its share of the host cores
if int(os.environ.get("WORLD_SIZE", "1")) > 1 or "OMP_NUM_THREADS" not in os.environ:
    os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 8) // int(os.environ.get("WORLD_SIZE", "1"))))

import numpy as np  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)  # BASELINE configs[4]: 200 steps
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg5", help="cfg1..cfg5 (default cfg5; N > 1: strong scaling of it)")
    ap.add_argument("--weak", action="store_true",
                    help="diagnostics: weak-scaling ladder at ~12.6 M tets per GPU instead of --config")
    ap.add_argument("--casting", type=int, default=0, help="diagnostics: an n^3-cell casting instead of a config")
    ap.add_argument("--mode", default="deterministic", choices=["atomic", "deterministic"])
    ap.add_argument("--tile", type=int, default=384)
    ap.add_argument("--elem-order", default="morton")
    ap.add_argument("--geometry", default="stored", choices=["stored", "coords"],
                    help="tile layout: slot coordinates (gradients recomputed) or stored ElementGeom")
    ap.add_argument("--node-order", default="tile",
                    help="the plan's local node numbering: tile (first touch in tile order, the B200 layout), "
                         "rcm (local ids in RCM label order) or given. cfg2's MESH is RCM-reordered (BASELINE "
                         "configs[1] 'RCM-reordered'): the generated mesh is renumbered by the device RCM pass "
                         "(permute_mesh(m, rcm_permutation(m))), in both arms; --mesh-rcm / --no-mesh-rcm override")
    ap.add_argument("--compare-order", default="rcm",
                    help="a second local numbering measured side by side (K steps, same mesh); 'none' to skip")
    ap.add_argument("--mesh-rcm", dest="mesh_rcm", action="store_true", default=None,
                    help="RCM-reorder the mesh (both arms); default: cfg2 only (the config that names it)")
    ap.add_argument("--no-mesh-rcm", dest="mesh_rcm", action="store_false")
    ap.add_argument("--cpu-steps", type=int, default=int(os.environ.get("CF_CPU_STEPS", "5")))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-blocked", action="store_true",
                    help="--impl reference: also time the reference's own cache blocking (autotune_block_count)")
    ap.add_argument("--ref-replicas", type=int, default=-1,
                    help="--impl reference: also run this many independent copies of the serial reference at once, "
                         "each pinned to its own core on its own 2-cell z-slab of the mesh (no exchange between "
                         "them): an upper bound for what the host's cores could do with a perfectly parallel "
                         "CPU run; -1 = one per core (default), 0 = skip")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", type=int, default=0, help="capture the step loop in CUDA graphs of this many steps")
    ap.add_argument("--phase-steps", type=int, default=20)
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer", "host", "peer-1gpu"],
                    help="N > 1: NCCL send/recv (one GPU per rank); peer = the pack kernel stores into the "
                         "neighbours' IPC windows over NVLink, streams wait on step flags (no library collective "
                         "on the data path); host = host-staged, every rank on cuda:0 (diagnostics); peer-1gpu = "
                         "the peer transport with every rank on cuda:0 (diagnostics)")
    return ap.parse_args()


def ncu_traffic(cfg: str, geometry: str, world: int):
    """DRAM bytes per tile-kernel launch from the committed ncu --set full capture of this
    workload and layout (profiles/ncu_traffic.json), else None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d["entries"][f"{cfg}/{geometry}"] if world == 1 else None
        return (int(e["traffic_bytes"]), "profiles/ncu_traffic.json") if e else (None, None)
    except (OSError, KeyError, ValueError):
        return None, None


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(
        os.environ.get("LOCAL_RANK", "0"))


def mesh_rcm_default(cfg: str, flag) -> bool:
    return (cfg == "cfg2") if flag is None else bool(flag)


def make_case(cfg: str, world: int, casting_n: int = 0, weak: bool = False, mesh_rcm: bool = False):
    from paper_1005_3158_b200 import configs
    if casting_n:
        return configs.casting(casting_n, dt_safety=configs.DT_SAFETY["cfg2"], steps=100,
                               name=f"casting{casting_n}"), f"casting{casting_n}", "weak"
    if weak and world > 1:
        n = int(round(128 * world ** (1.0 / 3.0)))
        return configs.casting(n, dt_safety=configs.DT_SAFETY["cfg4"], steps=500, name=f"casting{n}"), \
            f"weak_casting{n}", "weak"
    if cfg in ("cfg1", "cfg2", "cfg4", "cfg5") and not os.environ.get("CF_BENCH_HOST_MESH"):
        # the mesh is generated on the device (cf_plan_create_fixture): the same fixture and T0 as
        # the host-built case, without ~20 GB of host mesh per process at cfg5
        return configs.device_case(cfg, rcm=mesh_rcm), cfg, "strong" if world > 1 else "weak"
    return configs.CONFIGS[cfg](), cfg, "strong" if world > 1 else "weak"


# The reference arm's bounded sample per workload ("time a truncated run"). The
# reference needs ~420 B/tet of host memory and ~1.2 us/tet of setup: cfg5 in full
# would take > 300 GB and ~16 min, more than the GPU box's host (196 GB, 16 cores). The sample is a
# z-slab window of the SAME mesh -- same h, element shapes, regions, interface, initial field and
# dt -- with adiabatic cut planes: per-element work equals the full mesh's, so the per-element
# rate is the reference's rate on the workload. Full meshes where they fit in seconds.
REF_WINDOW = {"cfg4": [0, 256, 0, 256, 112, 144],   # 256 x 256 x 32 cells = 12,582,912 tets
              "cfg5": [0, 512, 0, 512, 252, 260]}   # 512 x 512 x 8 cells  = 12,582,912 tets
REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "ref_bench")


def reference_sample(cfg: str, steps: int, warmup: int, blocks: int = 1, autotune=None, window="default",
                     rcm: bool = False):
    """Runs the reference solver on the host (oracle/_ref/ref_bench, its own process: the
    unmodified castfem headers and the oracle's workload generator; no product library)."""
    if not os.path.exists(REF_BENCH):
        return None, "oracle/_ref/ref_bench not built (needs the reference headers at build time)"
    w = REF_WINDOW.get(cfg) if window == "default" else window
    cmd = [REF_BENCH, "--workload", cfg, "--steps", str(steps), "--warmup", str(warmup), "--blocks", str(blocks)]
    if w:
        cmd += ["--window", f"{w[0]}:{w[1]},{w[2]}:{w[3]},{w[4]}:{w[5]}"]
    if autotune:
        cmd += ["--autotune", ",".join(map(str, autotune))]
    if rcm:  # RCM-reordered mesh (the reference's own rcm_permutation + permute_mesh)
        cmd += ["--rcm"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        return None, f"ref_bench failed ({out.returncode}): {out.stderr.strip()[-300:]}"
    r = json.loads(out.stdout.strip().splitlines()[-1])
    what = (f"z-slab window cells {w[0]}:{w[1]} x {w[2]}:{w[3]} x {w[4]}:{w[5]} of the {cfg} mesh (same h, "
            f"regions, interface, T0 and dt; adiabatic cut planes)" if w else f"the full {cfg} mesh")
    what += ", RCM-reordered (the reference's rcm_permutation + permute_mesh)" if r.get("rcm") else ""
    r["sample"] = (f"{r['steps']} blocked_step calls after {r['warmup']} warm-up on {what}: E={r['elements']}, "
                   f"{r['blocks']} cache block(s); setup {r['setup_seconds']:.1f}s excluded (loop_seconds, "
                   f"blocked.hpp:673-684); serial by contract (SPEC S:403-408)")
    return r, None


def reference_replicas(cfg: str, steps: int, warmup: int, want: int):
    """`want` concurrent copies of the serial reference (ref_bench), each pinned to one core, each
    on its own 2-cell z-slab window of the cfg mesh (adiabatic cut planes, no exchange): the
    aggregate rate bounds from above what a perfectly parallel CPU run of the reference could reach
    on this host. Reported beside the 1-core figure; the reference itself is serial by contract."""
    n = {"cfg2": 128, "cfg4": 256, "cfg5": 512}.get(cfg)
    if n is None or not os.path.exists(REF_BENCH):
        return {"error": "replicas need a casting config and oracle/_ref/ref_bench"}
    cores = sorted(os.sched_getaffinity(0))
    P = len(cores) if want < 0 else min(want, len(cores))
    P = min(P, n // 2)
    try:  # ~1.5 GB per 2-cell slab of a 512^2 cross-section: stay well inside the free memory
        with open("/proc/meminfo") as f:
            avail_kb = next(int(l.split()[1]) for l in f if l.startswith("MemAvailable"))
        P = max(1, min(P, int(avail_kb / 1e6 / (2.0 * (n / 512.0) ** 2 + 0.2) / 2)))
    except Exception:
        P = min(P, 16)
    # slabs that cut the casting sphere (|z - 0.5| < 0.35), so every copy has both materials and
    # the interface; disjoint while P <= 0.33 n, as here
    lo, hi = int(0.16 * n) + 1, int(0.84 * n) - 3
    P = min(P, (hi - lo) // 2 + 1)
    procs = []
    for k in range(P):
        z0 = lo + (2 * (((hi - lo) // 2) * k // max(1, P - 1)) if P > 1 else (hi - lo) // 2)
        cmd = ["taskset", "-c", str(cores[k]), REF_BENCH, "--workload", cfg, "--steps", str(steps), "--warmup",
               str(warmup), "--blocks", "1", "--window", f"0:{n},0:{n},{z0}:{z0 + 2}"]
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    res = []
    for pr in procs:
        out, err = pr.communicate()
        if pr.returncode != 0:
            return {"error": f"ref_bench replica failed ({pr.returncode}): {err.strip()[-200:]}"}
        res.append(json.loads(out.strip().splitlines()[-1]))
    work = sum(r["elements"] * r["steps"] for r in res)
    slowest = max(r["seconds"] for r in res)
    return {"value": work / slowest, "unit": "element-updates/s", "cores": P, "kind": "reference",
            "sample": f"{P} concurrent copies of the serial reference, one per core (taskset), each {steps} "
                      f"blocked_step calls on its own 0:{n} x 0:{n} x 2-cell z-slab of the {cfg} mesh; total work / "
                      f"slowest copy's loop time; no exchange between copies (upper bound for a parallel CPU run)",
            "per_copy_min": min(r["element_updates_per_s"] for r in res),
            "per_copy_max": max(r["element_updates_per_s"] for r in res), "slowest_seconds": slowest}


def cpu_reference_rate(cfg: str, steps: int, rcm: bool = False):
    r, err = reference_sample(cfg, steps, 1, rcm=rcm)
    if r is None:
        return {"error": err}
    return {"value": r["element_updates_per_s"], "unit": "element-updates/s", "cores": 1, "kind": "reference",
            "sample": r["sample"], "seconds": r["seconds"]}


def _maps_product_library() -> bool:
    try:
        with open("/proc/self/maps") as f:
            return "libcastfem_b200" in f.read()
    except OSError:
        return False


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    steps, warmup = max(1, min(args.steps, 20)), min(args.warmup, 2)
    rcm = mesh_rcm_default(cfg, args.mesh_rcm)
    r, err = reference_sample(cfg, steps, warmup, rcm=rcm)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": err}), flush=True)
        return
    blocked = None
    if args.ref_blocked:  # the paper's technique: the reference's own cache blocking, autotuned
        b, berr = reference_sample(cfg, steps, warmup, autotune=[1, 16, 64, 256],
                                   window=[0, 512, 0, 512, 255, 257] if cfg == "cfg5" else "default",
                                   rcm=rcm)
        blocked = b if b is not None else {"error": berr}
    replicas = None
    if args.ref_replicas:  # reported beside the 1-core figure, never instead of it
        try:
            replicas = reference_replicas(cfg, steps, warmup, args.ref_replicas)
        except Exception as e:  # noqa: BLE001 -- an extra figure must not take the arm down
            replicas = {"error": f"{type(e).__name__}: {e}"}
    assert not _maps_product_library(), "the reference arm must not load the product library"
    value = r["element_updates_per_s"]
    line = {"impl": "reference", "metric": "element-updates/s (fp64)", "value": value, "unit": "element-updates/s",
            "n_gpus": 0, "steps": r["steps"], "warmup": r["warmup"], "ms_per_step": 1e3 * r["seconds"] / r["steps"],
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded Kuhn-split casting fixtures, SURVEY §8(d))",
            "config": {"workload": cfg, "sample_elements": r["elements"], "sample_nodes": r["nodes"],
                       "window": r["window"], "h_interface": 1000.0},
            "cpu_baseline": {"value": value, "unit": "element-updates/s", "cores": 1, "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": value, "unit": "element-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_run": {k: r[k] for k in ("seconds", "setup_seconds", "dt", "T_sum", "T_min", "T_max",
                                                "interface_pairs")},
            "reference_blocked": blocked, "reference_replicas": replicas}
    print(json.dumps(line), flush=True)


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML every 5 ms (the
    nvidia-smi CLI, ~100 ms per query, is the fallback)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, sm_max_mhz, set of active reason names)
        self.power_w = []  # board power under load (NVML only)
        self.power_limit_w = None
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nv = None

    def _one(self):
        if self._nv:
            nv, h = self._nv
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                        nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
                self.samples.append((float(sm), float(mx), {self.NAMES[i] for i, b in enumerate(bits) if r & b}))
                try:  # what sw_power_cap is capping against
                    self.power_w.append(nv.nvmlDeviceGetPowerUsage(h) / 1000.0)
                    if self.power_limit_w is None:
                        self.power_limit_w = nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
                except Exception:
                    pass
                return
            except Exception:
                self._nv = None
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            f = [x.strip() for x in out.stdout.strip().split(",")]
            if len(f) >= 7 and f[0].replace(".", "").isdigit():
                self.samples.append((float(f[0]), float(f[1]),
                                     {self.NAMES[i] for i in range(4) if f[3 + i] == "Active"}))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._one()
            self._stop.wait(0.005 if self._nv else 0.2)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            self._one()
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples]
        reasons = sorted(set().union(*[s[2] for s in self.samples])) if self.samples else []
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                # NVML's board power is a ~1 s moving average: over a short timed region it lags the load
                "power_w_max": round(max(self.power_w), 1) if self.power_w else None,
                "power_limit_w": self.power_limit_w,
                "source": "nvml" if self._nv else "nvidia-smi"}


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def main():
    args = parse()
    if "CF_PROBE" in os.environ:
        sys.exit("bench.py: CF_PROBE is a diagnostics knob (results invalid); unset it to measure")
    if args.impl == "reference":
        return run_reference(args)
    world, rank, local_rank = dist_env()
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist
        # launchers that isolate each rank with CUDA_VISIBLE_DEVICES show one device per process
        import torch
        ndev = torch.cuda.device_count()
        if ndev > 0:
            local_rank %= ndev
    from paper_1005_3158_b200 import castfem as cf

    mesh_rcm = mesh_rcm_default(args.config, args.mesh_rcm)
    case, cfg, scaling = make_case(args.config, world, args.casting, args.weak, mesh_rcm)
    setup = case.setup
    spec = getattr(case, "spec", None)  # device-generated mesh
    mesh = None if spec is not None else case.mesh
    comm = None
    if world > 1 and args.transport == "host":
        # diagnostics: several ranks on one GPU (NCCL refuses duplicate devices), exchange staged
        # through host memory over the gloo group; not a multi-GPU measurement
        local_rank = 0
        comm = cf.HostComm(world, rank, 0)
    elif world > 1 and args.transport in ("peer", "peer-1gpu"):
        if args.transport == "peer-1gpu":
            local_rank = 0
        comm = cf.PeerComm(world, rank, local_rank)
    elif world > 1:
        import torch
        # every rank must be able to load NCCL before anyone enters ncclCommInitRank (which waits
        # for all of them); if one cannot, all fall back to the host-staged transport, and say so
        try:
            uid = cf.Comm.unique_id()
            ok = 1
        except cf.CastfemError:
            uid, ok = bytes(128), 0
        flag = torch.tensor([ok], dtype=torch.int32)
        pg.all_reduce(flag, op=pg.ReduceOp.MIN)
        if int(flag[0]) == 1:
            t = torch.tensor(list(uid), dtype=torch.uint8)
            pg.broadcast(t, 0)
            comm = cf.Comm(world, rank, local_rank, bytes(t.tolist()))
        else:
            args.transport = "host (NCCL not loadable on every rank)"
            comm = cf.HostComm(world, rank, local_rank)
    opts = cf.SolveOptions(mode=args.mode, tile_elems=args.tile, elem_order=args.elem_order, geometry=args.geometry,
                           node_order=args.node_order, device=local_rank, world_size=world, rank=rank,
                           comm=comm, graph_steps=args.graph)
    t0 = time.time()
    solver = cf.Solver(mesh, setup, opts, fixture=spec)
    setup_s = time.time() - t0
    st0 = solver.stats()
    E_total = int(st0.n_elems_global)
    N_total = int(st0.n_nodes_global)
    T0_global = solver.fields(want_H=False)[0] if not args.no_e2e else None  # initial_temperatures

    def barrier():
        if pg:
            pg.barrier()

    def max_over_ranks(x: float) -> float:
        if not pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    # warm-up
    solver.step(max(args.warmup, 3))
    # timed region: K steps, device time (CUDA events), max over ranks
    sampler = ClockSampler(local_rank)
    barrier()
    sampler.start()
    before = solver.stats().loop_seconds
    solver.step(args.steps)
    secs = solver.stats().loop_seconds - before
    clocks = sampler.stop()
    secs = max_over_ranks(secs)
    barrier()
    value = E_total * args.steps / secs
    ms_per_step = 1e3 * secs / args.steps

    # per-phase device time (CUDA events between launches on the plan's stream)
    ph = solver.time_phases(args.phase_steps)
    st = solver.stats()
    N_local = st.n_nodes_local
    E_local = st.n_elems_local
    # algorithmic bytes of the tile (assembly) kernel per launch, DESIGN.md §roofline:
    # 105 B/tet (4 i32 conn + 11 f64 geometry + u8 region) + 24 B/node (T gather once,
    # (c, r) written once) + facets (canonical 24 / 56 B); the whole-step canonical
    # figure B_step = 105E + 48N + 24F_bc + 56F_if is st.bytes_per_step.
    # The coordinates layout reports its own bytes: blobs + slot T + outputs.
    facet_bytes = st.bytes_per_step - 105 * E_local - 48 * N_local
    if args.geometry == "stored":
        tile_bytes, bytes_model = 105 * E_local + 24 * N_local + facet_bytes, "canonical (SURVEY 8(d))"
    else:
        tile_bytes, bytes_model = st.tile_bytes_per_launch, "coordinates layout (blobs + slot T + outputs)"
    peak, peak_kind = hbm_peak()
    tile_gbs = tile_bytes / (ph[0] * 1e-3) / 1e9
    step_gbs = st.bytes_per_step / (ms_per_step * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(cfg, args.geometry, world)
    roofline = {"bound": "hbm", "kernel": "tile_kernel (assembly)", "achieved": round(tile_gbs, 1),
                "peak": peak, "unit": "GB/s", "frac": round(tile_gbs / peak, 4), "peak_kind": peak_kind,
                "traffic": traffic, "traffic_source": traffic_src, "bytes_model": bytes_model,
                "algorithmic_bytes_per_launch": int(tile_bytes),
                "kernel_ms": round(ph[0], 4), "update_ms": round(ph[3], 4), "pack_ms": round(ph[1], 4),
                "exchange_ms": round(ph[2], 4), "step_achieved_gbs": round(step_gbs, 1),
                "step_frac_of_8tbs": round(step_gbs / 8000.0, 4), "step_frac": round(step_gbs / peak, 4),
                "canonical_bytes_per_step": int(st.bytes_per_step),
                # the merge + update kernel's own byte model: per merged node its
                # record + T read/write, per partial the 16 B read + 8 B slot-copy write
                "update_kernel": {"algorithmic_bytes": int(st.update_bytes_per_step),
                                  "achieved_gbs": round(st.update_bytes_per_step / (ph[3] * 1e-3) / 1e9, 1)
                                  if ph[3] > 0 else None,
                                  "frac": round(st.update_bytes_per_step / (ph[3] * 1e-3) / 1e9 / peak, 4)
                                  if ph[3] > 0 else None}}

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        T0src = T0_global
        # pinned host buffers (the contract's host side): input T0, outputs T and H
        import torch
        pin = lambda: torch.empty(N_total, dtype=torch.float64, pin_memory=True).numpy()
        T0, Tout, Hout = pin(), pin(), pin()
        T0[:] = T0src
        # one untimed pass warms the path (first launches of the scatter / gather kernels load
        # them lazily; first transfers through freshly pinned pages)
        solver.set_temperature(T0)
        solver.step(1)
        solver.fields(out=(Tout, Hout))
        barrier()
        t1 = time.perf_counter()
        solver.set_temperature(T0)
        solver.step(args.steps)
        T, H = solver.fields(out=(Tout, Hout))
        e_secs = max_over_ranks(time.perf_counter() - t1)
        nb = N_total * 8
        e2e = {"value": E_total * args.steps / e_secs, "unit": "element-updates/s",
               "h2d_bytes_per_step": nb / args.steps, "d2h_bytes_per_step": 2 * nb / args.steps,
               "h2d_bytes_per_call": nb, "d2h_bytes_per_call": 2 * nb, "steps_per_call": args.steps,
               "seconds": e_secs, "host_buffers": "pinned",
               "api": "Solver.set_temperature -> Solver.step(K) -> Solver.fields()"}

    solver.close()
    # the other node ordering, side by side (node numbering leaves every result bitwise unchanged:
    # only the locality of the node arrays differs)
    order_cmp = None
    if args.compare_order not in ("none", "", args.node_order):
        o2 = cf.SolveOptions(**{**opts.__dict__, "node_order": args.compare_order})
        t2 = time.time()
        s2 = cf.Solver(mesh, setup, o2, fixture=spec)
        setup2 = time.time() - t2
        s2.step(max(args.warmup, 3))
        barrier()
        b2 = s2.stats().loop_seconds
        s2.step(args.steps)
        secs2 = max_over_ranks(s2.stats().loop_seconds - b2)
        ph2 = s2.time_phases(args.phase_steps)
        order_cmp = {"node_order": args.compare_order, "value": E_total * args.steps / secs2,
                     "ms_per_step": 1e3 * secs2 / args.steps, "kernel_ms": round(ph2[0], 4),
                     "update_ms": round(ph2[3], 4), "setup_seconds": round(setup2, 2)}
        s2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_rate(cfg, args.cpu_steps, rcm=mesh_rcm)
        except Exception as e:  # reported, not fatal
            cpu = {"error": str(e)}

    if rank == 0:
        line = {"metric": "element-updates/s (fp64)", "value": value, "unit": "element-updates/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded Kuhn-split casting fixtures, SURVEY §8(d))",
                "config": {"workload": cfg, "elements": E_total, "nodes": N_total,
                           "mesh_source": "generated on the device (cf_plan_create_fixture)" if spec is not None
                           else "host arrays (cf_plan_create)",
                           "mesh_numbering": "RCM (device pass: permute_mesh(m, rcm_permutation(m)))"
                           if spec is not None and spec.rcm else "generator",
                           "hex_cells": E_total // 6, "mode": args.mode, "tile_elems": args.tile,
                           "elem_order": args.elem_order, "node_order": args.node_order,
                           "geometry": args.geometry,
                           "dt_safety": setup.solver.dt_safety, "h_interface": 1000.0,
                           "parallelism": f"rcb{world}" if world > 1 else "single",
                           "transport": (args.transport if world > 1 else None),
                           "setup_pipeline": "device" if st0.device_setup else "host",
                           "l2": "working set > 126 MB L2 (no flush needed)" if st.bytes_per_step > 2e8
                           else "working set L2-resident", "setup_seconds": round(setup_s, 2)},
                "hex_cell_updates_per_s": value / 6.0,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(st.launches_per_step * args.steps), "clocks": clocks,
                "device_bytes": int(st.device_bytes), "tiles": int(st.n_tiles),
                "host_peak_rss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20, 2),
                "total_slots": int(st.total_slots),
                "env": {k: v for k, v in sorted(os.environ.items()) if k.startswith("CF_")},
                "build": "production (probe branches compiled out: no CF_DIAG)",
                "node_order_comparison": order_cmp}
        print(json.dumps(line), flush=True)
    if comm:
        comm.close()
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
