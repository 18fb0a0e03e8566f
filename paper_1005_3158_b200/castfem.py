"""Python mirror of the reference castfem C++ API, running on the B200 path.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/castfem/, cited relative to that directory):

  Mesh                 mesh.hpp:45-80         (nodes / tets / facets / tags / contacts)
  PiecewiseLinear      material.hpp:21-47
  MaterialTable        material.hpp:53-124
  BoundaryCondition    material.hpp:126-141   (kind 'fixed' | 'flux')
  InterfaceCoeff       material.hpp:145-153   (var 'time' | 'temperature')
  SolverConfig         material.hpp:155-160
  SimulationSetup      material.hpp:162-184   (initial_T replaces the initial_override hook)
  SolveOptions         blocked.hpp:630-636    (+ B200 tiling / mode / decomposition options)
  SolveResult          blocked.hpp:638-647
  solve_serial         blocked.hpp:650-696    -> solve() on the GPU
  Solver               build_worker_model + init_worker_fields + blocked_step granularity
  rcm_permutation, bandwidth, permute_mesh      reorder.hpp:41-163
  finalize_mesh, pair_sister_facets             mesh.hpp:148-207, 456-478
  exceptions           errors.hpp:8-31 (+ DegenerateElementError geometry.hpp:43-46)

Every compute call goes through the C-ABI in include/castfem_b200.h into
libcastfem_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from ._abi import lib


# ------------------------------------------------------------------ errors (errors.hpp)
class CastfemError(RuntimeError):
    code = -1


class ParseError(CastfemError):
    code = _abi.CF_PARSE


class ValidationError(CastfemError):
    code = _abi.CF_VALIDATION


class ConfigError(CastfemError):
    code = _abi.CF_CONFIG


class ProtocolError(CastfemError):
    code = _abi.CF_PROTOCOL


class DegenerateElementError(CastfemError):
    code = _abi.CF_DEGENERATE


class CudaError(CastfemError):
    code = _abi.CF_CUDA


class NcclError(CastfemError):
    code = _abi.CF_NCCL


class InvalidArgument(CastfemError, ValueError):
    code = _abi.CF_INVALID_ARG


_BY_CODE = {c.code: c for c in (ParseError, ValidationError, ConfigError, ProtocolError, DegenerateElementError,
                                CudaError, NcclError, InvalidArgument)}


def check(status: int) -> None:
    if status != _abi.CF_OK:
        raise _BY_CODE.get(status, CastfemError)(_abi.last_error())


# ------------------------------------------------------------------ model types
@dataclass
class PiecewiseLinear:
    xs: List[float] = field(default_factory=list)
    ys: List[float] = field(default_factory=list)

    @staticmethod
    def constant(v: float) -> "PiecewiseLinear":
        return PiecewiseLinear([0.0], [float(v)])

    def is_constant(self) -> bool:
        return len(self.xs) <= 1


def _pl(v) -> PiecewiseLinear:
    if isinstance(v, PiecewiseLinear):
        return v
    if isinstance(v, (int, float)):
        return PiecewiseLinear.constant(float(v))
    xs, ys = zip(*v)
    return PiecewiseLinear(list(map(float, xs)), list(map(float, ys)))


@dataclass
class MaterialTable:
    rho: float = 0.0
    c_of_T: PiecewiseLinear = field(default_factory=PiecewiseLinear)
    k_of_T: PiecewiseLinear = field(default_factory=PiecewiseLinear)
    latent_heat: float = 0.0
    solidus: float = 0.0
    liquidus: float = 0.0
    initial_temperature: float = 0.0

    @staticmethod
    def make(rho, c, k, latent_heat=0.0, solidus=0.0, liquidus=0.0, T0=0.0) -> "MaterialTable":
        return MaterialTable(float(rho), _pl(c), _pl(k), float(latent_heat), float(solidus), float(liquidus),
                             float(T0))


@dataclass
class BoundaryCondition:
    kind: str = "flux"  # 'fixed' | 'flux'
    fixed_T: PiecewiseLinear = field(default_factory=PiecewiseLinear)
    q: float = 0.0
    h: float = 0.0
    t_inf: float = 0.0


@dataclass
class InterfaceCoeff:
    tag_a: str
    tag_b: str
    var: str = "time"  # 'time' | 'temperature'
    h: PiecewiseLinear = field(default_factory=lambda: PiecewiseLinear.constant(0.0))


@dataclass
class SolverConfig:
    dt_safety: float = 0.5
    t_end: float = 0.0
    output_every: int = 0


@dataclass
class SimulationSetup:
    materials: List[MaterialTable] = field(default_factory=list)
    boundary_conditions: Dict[str, BoundaryCondition] = field(default_factory=dict)
    interface_coeffs: List[InterfaceCoeff] = field(default_factory=list)
    solver: SolverConfig = field(default_factory=SolverConfig)
    initial_T: Optional[np.ndarray] = None  # index-keyed initial field (initial_override analogue)


@dataclass
class Mesh:
    nodes: np.ndarray        # (N, 3) float64
    tets: np.ndarray         # (E, 4) int32
    region: np.ndarray       # (E,) int32
    facets: np.ndarray       # (F, 3) int32
    facet_tag: np.ndarray    # (F,) int32
    tags: List[str]
    contacts: List[Tuple[int, int]] = field(default_factory=list)
    node_grid: Optional[np.ndarray] = None  # fixtures: grid point of each node

    def __post_init__(self):
        self.nodes = np.ascontiguousarray(self.nodes, dtype=np.float64).reshape(-1, 3)
        self.tets = np.ascontiguousarray(self.tets, dtype=np.int32).reshape(-1, 4)
        self.region = np.ascontiguousarray(self.region, dtype=np.int32).reshape(-1)
        self.facets = np.ascontiguousarray(self.facets, dtype=np.int32).reshape(-1, 3)
        self.facet_tag = np.ascontiguousarray(self.facet_tag, dtype=np.int32).reshape(-1)

    def node_count(self) -> int:
        return int(self.nodes.shape[0])

    def element_count(self) -> int:
        return int(self.tets.shape[0])

    def tag_id(self, name: str) -> int:
        return self.tags.index(name) if name in self.tags else -1


@dataclass
class SolveOptions:
    """SolveOptions (blocked.hpp:630-636) + the B200 knobs."""
    max_steps: int = 0
    mode: str = "deterministic"      # 'deterministic' (bit-reproducible, fastest) | 'atomic' (fp64 RED)
    node_order: str = "tile"         # 'tile' (first touch in tile order) | 'rcm' | 'given'
    elem_order: str = "morton"       # 'morton' | 'min_node' | 'given'
    tile_elems: int = 384
    geometry: str = "stored"         # 'stored' (ElementGeom per tet) | 'coords' (recompute from slot coordinates)
    blocks: Optional[np.ndarray] = None  # explicit element->tile map (BlockPlan semantics)
    device: int = 0
    world_size: int = 1
    rank: int = 0
    local_ranks: int = 1
    part_of_element: Optional[np.ndarray] = None
    partition: str = "rcb"           # 'rcb' | 'graph' (virtual-element augmented greedy partitioner)
    comm: Optional["Comm"] = None    # Comm (NCCL) or HostComm (host-staged) for world_size > local_ranks
    graph_steps: int = 0


@dataclass
class SeriesSample:
    time: float
    t_min: float
    t_max: float


@dataclass
class SolveResult:
    T: np.ndarray
    H: np.ndarray
    end_time: float
    steps: int
    loop_seconds: float
    series: List[SeriesSample]
    clamp_steps: int
    blocks_used: int


# ------------------------------------------------------------------ descriptors
class _Keep:
    """Holds the numpy buffers a descriptor points into."""

    def __init__(self):
        self.refs = []

    def arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.refs.append(a)
        return a

    def dptr(self, a):
        a = self.arr(a, np.float64)
        return a.ctypes.data_as(C.POINTER(C.c_double))

    def iptr(self, a):
        a = self.arr(a, np.int32)
        return a.ctypes.data_as(C.POINTER(C.c_int32))

    def table(self, t: PiecewiseLinear) -> _abi.cf_table:
        n = len(t.xs)
        if n == 0:
            return _abi.cf_table(0, None, None)
        return _abi.cf_table(n, self.dptr(t.xs), self.dptr(t.ys))

    def cstr(self, s: str):
        b = s.encode()
        self.refs.append(b)
        return b


def mesh_desc(m: Mesh, keep: _Keep) -> _abi.cf_mesh_desc:
    d = _abi.cf_mesh_desc()
    d.n_nodes = m.node_count()
    d.coords = keep.dptr(m.nodes)
    d.n_elems = m.element_count()
    d.tets = keep.iptr(m.tets)
    d.region = keep.iptr(m.region)
    d.n_facets = int(m.facets.shape[0])
    d.facets = keep.iptr(m.facets)
    d.facet_tag = keep.iptr(m.facet_tag)
    d.n_tags = len(m.tags)
    tags = (C.c_char_p * max(1, len(m.tags)))(*[keep.cstr(t) for t in m.tags])
    keep.refs.append(tags)
    d.tags = C.cast(tags, C.POINTER(C.c_char_p))
    d.n_contacts = len(m.contacts)
    d.contacts = keep.iptr(np.array(m.contacts, dtype=np.int32).reshape(-1) if m.contacts else np.zeros(2, np.int32))
    return d


def setup_desc(s: SimulationSetup, keep: _Keep) -> _abi.cf_setup_desc:
    d = _abi.cf_setup_desc()
    mats = (_abi.cf_material * max(1, len(s.materials)))()
    for i, m in enumerate(s.materials):
        mats[i] = _abi.cf_material(m.rho, keep.table(m.c_of_T), keep.table(m.k_of_T), m.latent_heat, m.solidus,
                                   m.liquidus, m.initial_temperature)
    keep.refs.append(mats)
    bcs = (_abi.cf_boundary_condition * max(1, len(s.boundary_conditions)))()
    for i, (tag, b) in enumerate(s.boundary_conditions.items()):
        kind = _abi.CF_BC_FIXED if b.kind == "fixed" else _abi.CF_BC_FLUX
        bcs[i] = _abi.cf_boundary_condition(keep.cstr(tag), kind, keep.table(b.fixed_T), b.q, b.h, b.t_inf)
    keep.refs.append(bcs)
    cos = (_abi.cf_interface_coeff * max(1, len(s.interface_coeffs)))()
    for i, c in enumerate(s.interface_coeffs):
        var = _abi.CF_VAR_TEMPERATURE if c.var == "temperature" else _abi.CF_VAR_TIME
        cos[i] = _abi.cf_interface_coeff(keep.cstr(c.tag_a), keep.cstr(c.tag_b), var, keep.table(c.h))
    keep.refs.append(cos)
    d.n_materials = len(s.materials)
    d.materials = mats
    d.n_bcs = len(s.boundary_conditions)
    d.bcs = bcs
    d.n_coeffs = len(s.interface_coeffs)
    d.coeffs = cos
    d.dt_safety = s.solver.dt_safety
    d.t_end = s.solver.t_end
    d.output_every = int(s.solver.output_every)
    d.initial_T = keep.dptr(s.initial_T) if s.initial_T is not None else None
    return d


_MODES = {"atomic": _abi.CF_MODE_ATOMIC, "deterministic": _abi.CF_MODE_DETERMINISTIC}
_NODE = {"given": _abi.CF_NODE_ORDER_GIVEN, "rcm": _abi.CF_NODE_ORDER_RCM, "tile": _abi.CF_NODE_ORDER_TILE}
_ELEM = {"given": _abi.CF_ELEM_ORDER_GIVEN, "morton": _abi.CF_ELEM_ORDER_MORTON,
         "min_node": _abi.CF_ELEM_ORDER_MIN_NODE}
_GEOM = {"coords": _abi.CF_GEOM_COORDS, "stored": _abi.CF_GEOM_STORED}


def run_opts(o: SolveOptions, keep: _Keep) -> _abi.cf_run_opts:
    d = _abi.cf_run_opts()
    d.device = o.device
    d.mode = _MODES[o.mode]
    d.node_order = _NODE[o.node_order]
    d.elem_order = _ELEM[o.elem_order]
    d.tile_elems = o.tile_elems
    d.geometry = _GEOM[o.geometry]
    if o.blocks is not None:
        d.tile_of_element = keep.iptr(o.blocks)
        d.n_tiles_given = int(np.max(o.blocks)) + 1 if len(o.blocks) else 0
    d.world_size = o.world_size
    d.rank = o.rank
    d.local_ranks = o.local_ranks
    if o.part_of_element is not None:
        d.partition = _abi.CF_PARTITION_GIVEN
        d.part_of_element = keep.iptr(o.part_of_element)
    elif o.partition == "graph":
        d.partition = _abi.CF_PARTITION_GRAPH
    d.comm = o.comm.handle if o.comm is not None else None
    return d


# ------------------------------------------------------------------ multi-rank
class Comm:
    """NCCL communicator (one rank per GPU). Rank 0 creates the unique id."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().cf_comm_unique_id(buf))
        return buf.raw

    def __init__(self, world_size: int, rank: int, device: int, uid: bytes):
        h = C.c_void_p()
        check(lib().cf_comm_create(world_size, rank, device, uid, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib().cf_comm_destroy(self.handle)
            self.handle = None


class HostComm:
    """Host-staged transport (cf_comm_create_host): the per-step exchange_and_merge payload
     and the per-rank scalar reductions go through a torch.distributed process
    group (e.g. gloo) instead of NCCL -- for rank processes that share one GPU (NCCL refuses
    duplicate devices) or hosts without a GPU interconnect. One paired send/recv round per step
    with every neighbour, like the NCCL path."""

    def __init__(self, world_size: int, rank: int, device: int, group=None):
        import torch
        import torch.distributed as dist
        self._dist, self._torch, self._group = dist, torch, group

        def sendrecv(ctx, n, peers, send, send_len, recv, recv_len):
            try:
                reqs = []
                for k in range(n):
                    q = int(peers[k])
                    if send_len[k]:
                        buf = np.ctypeslib.as_array(send[k], shape=(int(send_len[k]),))
                        reqs.append(dist.isend(torch.from_numpy(buf), q, group=group))
                    if recv_len[k]:
                        buf = np.ctypeslib.as_array(recv[k], shape=(int(recv_len[k]),))
                        reqs.append(dist.irecv(torch.from_numpy(buf), q, group=group))
                for r in reqs:
                    r.wait()
                return 0
            except Exception:  # reported by the library as CF_PROTOCOL
                return 1

        def allreduce(ctx, values, n, op):
            try:
                buf = np.ctypeslib.as_array(values, shape=(int(n),))
                t = torch.from_numpy(buf)
                dist.all_reduce(t, op=dist.ReduceOp.MIN if op == _abi.CF_REDUCE_MIN else dist.ReduceOp.MAX,
                                group=group)
                return 0
            except Exception:
                return 1

        # the callbacks must outlive the communicator
        self._cb = (_abi.SENDRECV_FN(sendrecv), _abi.ALLREDUCE_FN(allreduce))
        t = _abi.cf_host_transport(None, self._cb[0], self._cb[1])
        h = C.c_void_p()
        check(getattr(lib(), self._create)(world_size, rank, device, C.byref(t), C.byref(h)))
        self.handle = h

    _create = "cf_comm_create_host"

    def close(self):
        if self.handle:
            lib().cf_comm_destroy(self.handle)
            self.handle = None


class PeerComm(HostComm):
    """Peer-memory transport (cf_comm_create_peer): the pack kernel stores each neighbour's
    payload straight into that neighbour's IPC-exported device window over NVLink and raises a
    step flag the neighbour's stream waits on; no library collective on the data path. The
    torch.distributed group (gloo is enough) only carries the one-time window-handle exchange
    and the barrier at plan destruction. Close the Solver before this communicator."""

    _create = "cf_comm_create_peer"


# ------------------------------------------------------------------ solver
class Solver:
    """A device-resident plan: build_worker_model + init_worker_fields
    (blocked.hpp:156-436), stepped with blocked_step semantics (:542-550)."""

    def __init__(self, mesh: Optional[Mesh], setup: SimulationSetup, opts: Optional[SolveOptions] = None,
                 fixture: Optional["FixtureSpec"] = None):
        """mesh: host arrays (cf_plan_create); or fixture: the mesh generated on the device
        (cf_plan_create_fixture: it never exists in host memory)."""
        opts = opts or SolveOptions()
        keep = _Keep()
        self.mesh = mesh
        self.setup = setup
        self.opts = opts
        sd, ro = setup_desc(setup, keep), run_opts(opts, keep)
        h = C.c_void_p()
        if (mesh is None) == (fixture is None):
            raise InvalidArgument("Solver needs exactly one of mesh (host arrays) or fixture (device-generated)")
        if fixture is not None:
            fx = fixture.desc()
            check(lib().cf_plan_create_fixture(C.byref(fx), C.byref(sd), C.byref(ro), C.byref(h)))
        else:
            md = mesh_desc(mesh, keep)
            check(lib().cf_plan_create(C.byref(md), C.byref(sd), C.byref(ro), C.byref(h)))
        self.handle = h
        self._N = int(self.stats().n_nodes_global)
        if opts.graph_steps:
            check(lib().cf_enable_graph(self.handle, opts.graph_steps))

    # --- state
    def set_temperature(self, T: np.ndarray) -> None:
        T = np.ascontiguousarray(T, dtype=np.float64)
        if T.shape != (self._N,):
            raise InvalidArgument("temperature field must have one value per node")
        check(lib().cf_set_temperature(self.handle, T.ctypes.data_as(C.POINTER(C.c_double))))

    def set_dt_safety(self, s: float) -> None:
        check(lib().cf_set_dt_safety(self.handle, float(s)))

    def step(self, n: int = 1, t_end: float = 0.0) -> None:
        check(lib().cf_step(self.handle, int(n), float(t_end)))

    def solve(self, max_steps: int = 0) -> List[SeriesSample]:
        cap = 1 << 16
        buf = np.zeros(3 * cap)
        n = C.c_int64()
        check(lib().cf_solve(self.handle, int(max_steps), buf.ctypes.data_as(C.POINTER(C.c_double)), cap,
                             C.byref(n)))
        k = min(n.value, cap)
        return [SeriesSample(*buf[3 * i:3 * i + 3]) for i in range(k)]

    def fields(self, want_H: bool = True, out: Optional[Tuple[np.ndarray, Optional[np.ndarray]]] = None
               ) -> Tuple[np.ndarray, Optional[np.ndarray]]:
        """Global-order T (and H). `out` = caller-owned float64 arrays of node_count() entries
        (e.g. pinned host memory) filled in place."""
        if out is not None:
            T, H = out
            for a in (T, H):
                if a is not None and (a.dtype != np.float64 or not a.flags.c_contiguous or a.size != self._N):
                    raise ValueError("fields(out=...) needs C-contiguous float64 arrays of node_count() entries")
            if not want_H:
                H = None
        else:
            T = np.zeros(self._N)
            H = np.zeros(self._N) if want_H else None
        check(lib().cf_get_fields(self.handle, T.ctypes.data_as(C.POINTER(C.c_double)),
                                  H.ctypes.data_as(C.POINTER(C.c_double)) if want_H else None))
        return T, H

    def stats(self) -> _abi.cf_stats:
        s = _abi.cf_stats()
        check(lib().cf_get_stats(self.handle, C.byref(s)))
        return s

    def time_phases(self, n: int) -> np.ndarray:
        """n real steps with CUDA events between phases: mean ms of (tile, pack, exchange, update)."""
        out = np.zeros(4)
        check(lib().cf_time_phases(self.handle, int(n), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def enable_graph(self, steps: int) -> None:
        check(lib().cf_enable_graph(self.handle, int(steps)))

    def device_temperature(self, local_rank: int = 0) -> Tuple[int, int]:
        p = C.POINTER(C.c_double)()
        n = C.c_int64()
        check(lib().cf_device_temperature(self.handle, local_rank, C.byref(p), C.byref(n)))
        return C.cast(p, C.c_void_p).value, n.value

    def estimate_lambda_max(self, iterations: int = 500, seed: int = 1234) -> Tuple[float, float]:
        lam, e13 = C.c_double(), C.c_double()
        check(lib().cf_estimate_lambda_max(self.handle, int(iterations), int(seed), C.byref(lam), C.byref(e13)))
        return lam.value, e13.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().cf_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def solve(mesh: Mesh, setup: SimulationSetup, opts: Optional[SolveOptions] = None) -> SolveResult:
    """solve_serial (blocked.hpp:650-696) on the B200: same loop semantics
    (max_steps, or run to setup.solver.t_end), same SolveResult fields;
    loop_seconds is device time of the step loop (setup excluded)."""
    opts = opts or SolveOptions()
    with Solver(mesh, setup, opts) as s:
        series = s.solve(opts.max_steps)
        T, H = s.fields()
        st = s.stats()
        return SolveResult(T, H, st.time, st.step_index, st.loop_seconds, series, st.clamp_steps, st.n_tiles)


solve_serial = solve


# ------------------------------------------------------------------ host utilities
def finalize_mesh(m: Mesh) -> Tuple[np.ndarray, np.ndarray]:
    """finalize_mesh (mesh.hpp:148-207): returns (oriented tets, facet owners)."""
    keep = _Keep()
    d = mesh_desc(m, keep)
    tets = np.zeros((m.element_count(), 4), np.int32)
    owner = np.zeros(max(1, m.facets.shape[0]), np.int32)
    check(lib().cf_finalize_mesh(C.byref(d), tets.ctypes.data_as(C.POINTER(C.c_int32)),
                                 owner.ctypes.data_as(C.POINTER(C.c_int32))))
    return tets, owner[:m.facets.shape[0]]


def pair_sister_facets(m: Mesh) -> np.ndarray:
    """pair_sister_facets (mesh.hpp:456-478): (P, 3) rows (facet, sister, contact)."""
    keep = _Keep()
    d = mesh_desc(m, keep)
    n = C.c_int64()
    check(lib().cf_pair_sister_facets(C.byref(d), None, 0, C.byref(n)))
    out = np.zeros((max(1, n.value), 3), np.int32)
    check(lib().cf_pair_sister_facets(C.byref(d), out.ctypes.data_as(C.POINTER(C.c_int32)), n.value, C.byref(n)))
    return out[:n.value]


def rcm_permutation(m: Mesh, seed: int = -1) -> np.ndarray:
    """rcm_permutation(build_node_graph(m)) (reorder.hpp:17-24, 127-148): new_of_old."""
    keep = _Keep()
    d = mesh_desc(m, keep)
    out = np.zeros(m.node_count(), np.int32)
    check(lib().cf_rcm_permutation(C.byref(d), int(seed), out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def rcm_permutation_device(m: Mesh, seed: int = -1, device: int = 0) -> np.ndarray:
    """The same permutation computed on the B200 (the plan builder's RCM pass, cf_rcm.cu)."""
    keep = _Keep()
    d = mesh_desc(m, keep)
    out = np.zeros(m.node_count(), np.int32)
    check(lib().cf_rcm_permutation_device(C.byref(d), int(seed), int(device), out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def bandwidth(m: Mesh, new_of_old: Optional[np.ndarray] = None) -> int:
    keep = _Keep()
    d = mesh_desc(m, keep)
    out = C.c_int64()
    p = keep.iptr(new_of_old) if new_of_old is not None else None
    check(lib().cf_bandwidth(C.byref(d), p, C.byref(out)))
    return out.value


def permute_mesh(m: Mesh, new_of_old: np.ndarray) -> Mesh:
    """permute_mesh (reorder.hpp:152-163): renumbers nodes only."""
    p = np.asarray(new_of_old, dtype=np.int64)
    if p.shape[0] != m.node_count():
        raise ValidationError(f"permutation size {p.shape[0]} does not match node count {m.node_count()}")
    nodes = np.empty_like(m.nodes)
    nodes[p] = m.nodes
    ng = None
    if m.node_grid is not None:
        ng = np.empty_like(m.node_grid)
        ng[p] = m.node_grid
    return Mesh(nodes, p[m.tets].astype(np.int32), m.region.copy(), p[m.facets].astype(np.int32),
                m.facet_tag.copy(), list(m.tags), list(m.contacts), ng)


def partition_rcb(m: Mesh, parts: int) -> np.ndarray:
    keep = _Keep()
    d = mesh_desc(m, keep)
    out = np.zeros(m.element_count(), np.int32)
    check(lib().cf_partition_rcb(C.byref(d), int(parts), out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def partition_elements(m: Mesh, parts: int, balance_tol: float = 0.05, augment: bool = True) -> np.ndarray:
    """Graph partition of the elements (partition_graph partition.hpp:134-232 over the dual graph,
    augmented with virtual elements across interface pairs when `augment`)."""
    keep = _Keep()
    d = mesh_desc(m, keep)
    out = np.zeros(m.element_count(), np.int32)
    check(lib().cf_partition_graph(C.byref(d), int(parts), float(balance_tol), int(bool(augment)),
                                   out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


@dataclass
class PartitionQuality:
    edge_cut: int
    imbalance: float
    neighbor_counts: List[int]
    split_interface_pairs: int


def partition_metrics(m: Mesh, parts_of_element: np.ndarray, parts: int) -> PartitionQuality:
    """partition_metrics + count_split_interface_pairs (partition.hpp:250-283)."""
    keep = _Keep()
    d = mesh_desc(m, keep)
    cut, split = C.c_int64(), C.c_int64()
    imb = C.c_double()
    nb = np.zeros(max(1, parts), np.int32)
    check(lib().cf_partition_metrics(C.byref(d), keep.iptr(parts_of_element), int(parts), C.byref(cut), C.byref(imb),
                                     nb.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(split)))
    return PartitionQuality(cut.value, imb.value, nb[:parts].tolist(), split.value)


def tile_map(m: Mesh, setup: SimulationSetup, opts: SolveOptions) -> Tuple[np.ndarray, int]:
    """Element -> tile map the plan would build (the BlockPlan the oracle replays)."""
    keep = _Keep()
    md, sd, ro = mesh_desc(m, keep), setup_desc(setup, keep), run_opts(opts, keep)
    out = np.zeros(m.element_count(), np.int32)
    n = C.c_int32()
    check(lib().cf_tile_map(C.byref(md), C.byref(sd), C.byref(ro), out.ctypes.data_as(C.POINTER(C.c_int32)),
                            C.byref(n)))
    return out, n.value


DIGEST_NAMES = ("scalars", "tile_meta", "tile_border", "tile_slot_off", "blob_off", "elem_off", "blob_staged",
                "tets_ord", "elem_global", "slot_node", "local_global", "node_region", "node_dir", "merge_off",
                "merge_idx", "shared_list", "neighbors", "exchange")


def plan_digest(m: Mesh, setup: SimulationSetup, opts: SolveOptions, rank: int = 0, device: bool = False) -> dict:
    """Per-array digests of one rank's tiled plan from the host plan builder, or (device=True)
    from the device setup pipeline (test instrumentation: the two must agree)."""
    keep = _Keep()
    md, sd, ro = mesh_desc(m, keep), setup_desc(setup, keep), run_opts(opts, keep)
    out = (C.c_uint64 * 24)()
    fn = lib().cf_plan_digest_device if device else lib().cf_plan_digest
    check(fn(C.byref(md), C.byref(sd), C.byref(ro), rank, out))
    return {k: int(out[i]) for i, k in enumerate(DIGEST_NAMES)}


def partition_rcb_device(m: Mesh, parts: int) -> np.ndarray:
    """partition_rcb computed on the B200 (equal to partition_rcb)."""
    keep = _Keep()
    md = mesh_desc(m, keep)
    out = np.zeros(m.element_count(), np.int32)
    check(lib().cf_partition_rcb_device(C.byref(md), int(parts), out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


@dataclass
class FixtureSpec:
    """A structured fixture generated on the device (generate_fixture with perm_seed 0), and
    its T0 rule: region T0 + U(-t0_noise, t0_noise) keyed by grid point (counter_uniform)."""
    kind: str = "casting"
    n: int = 32
    radius: float = 0.35
    jitter: float = 0.0
    seed: int = 0
    t0_noise: float = 0.0
    noise_seed: int = 1
    rcm: bool = False       # node numbering permuted by the RCM pass (an RCM-reordered mesh)

    def desc(self) -> "_abi.cf_fixture_spec":
        return _abi.cf_fixture_spec({"cube": 0, "casting": 1}[self.kind], int(self.n), float(self.radius),
                                    float(self.jitter), int(self.seed), 0, float(self.t0_noise), int(self.noise_seed),
                                    int(self.rcm))

    def mesh(self) -> Mesh:
        """The same mesh on the host (cf_generate_fixture, then permute_mesh by rcm_permutation)."""
        m = generate_fixture(self.kind, self.n, radius=self.radius, jitter=self.jitter, seed=self.seed)
        return permute_mesh(m, rcm_permutation(m)) if self.rcm else m


def exchange_plan(m: Mesh, setup: SimulationSetup, world_size: int, rank: int,
                  part_of_element: Optional[np.ndarray] = None) -> List[dict]:
    """Rank `rank`'s neighbours and exchange lists (global node ids): shared
    nodes (c, r partials travel in this order) and external nodes whose
    pre-update T flows to / from each neighbour."""
    keep = _Keep()
    md, sd = mesh_desc(m, keep), setup_desc(setup, keep)
    ro = run_opts(SolveOptions(world_size=world_size, rank=rank, part_of_element=part_of_element), keep)
    nn = C.c_int32()
    check(lib().cf_exchange_plan(C.byref(md), C.byref(sd), C.byref(ro), C.byref(nn), None, None, None, None, None))
    k = nn.value
    ranks = np.zeros(max(k, 1), np.int32)
    counts = np.zeros(3 * max(k, 1), np.int64)
    check(lib().cf_exchange_plan(C.byref(md), C.byref(sd), C.byref(ro), C.byref(nn),
                                 ranks.ctypes.data_as(C.POINTER(C.c_int32)),
                                 counts.ctypes.data_as(C.POINTER(C.c_int64)), None, None, None))
    tot = counts.reshape(-1, 3)[:k].sum(0) if k else np.zeros(3, np.int64)
    sh, to, fr = (np.zeros(max(1, int(t)), np.int32) for t in tot)
    check(lib().cf_exchange_plan(C.byref(md), C.byref(sd), C.byref(ro), C.byref(nn), None, None,
                                 sh.ctypes.data_as(C.POINTER(C.c_int32)), to.ctypes.data_as(C.POINTER(C.c_int32)),
                                 fr.ctypes.data_as(C.POINTER(C.c_int32))))
    out, a, b, c = [], 0, 0, 0
    for j in range(k):
        ns, nt, nf = (int(x) for x in counts[3 * j:3 * j + 3])
        out.append({"rank": int(ranks[j]), "shared": sh[a:a + ns].copy(), "ext_to": to[b:b + nt].copy(),
                    "ext_from": fr[c:c + nf].copy()})
        a, b, c = a + ns, b + nt, c + nf
    return out


def generate_fixture(kind: str, n: int, radius: float = 0.35, jitter: float = 0.0, seed: int = 0,
                     perm_seed: int = 0) -> Mesh:
    """Structured Kuhn 6-tet fixtures (SPEC bench module S:502-519): 'cube' or 'casting'."""
    k = {"cube": 0, "casting": 1}[kind]
    fx = _abi.cf_fixture()
    check(lib().cf_generate_fixture(k, n, radius, jitter, seed, perm_seed, C.byref(fx)))
    N, E, F = fx.n_nodes, fx.n_elems, fx.n_facets
    coords = np.zeros((N, 3))
    tets = np.zeros((E, 4), np.int32)
    region = np.zeros(E, np.int32)
    facets = np.zeros((max(F, 1), 3), np.int32)
    ftag = np.zeros(max(F, 1), np.int32)
    grid = np.zeros(N, np.int32)
    fx.coords = coords.ctypes.data_as(C.POINTER(C.c_double))
    fx.tets = tets.ctypes.data_as(C.POINTER(C.c_int32))
    fx.region = region.ctypes.data_as(C.POINTER(C.c_int32))
    fx.facets = facets.ctypes.data_as(C.POINTER(C.c_int32))
    fx.facet_tag = ftag.ctypes.data_as(C.POINTER(C.c_int32))
    fx.node_grid = grid.ctypes.data_as(C.POINTER(C.c_int32))
    check(lib().cf_generate_fixture(k, n, radius, jitter, seed, perm_seed, C.byref(fx)))
    tags = ["outer", "cast_if", "mold_if"] if k == 1 else ["outer"]
    contacts = [(1, 2)] if k == 1 else []
    return Mesh(coords, tets, region, facets[:F], ftag[:F], tags, contacts, grid)


def counter_uniform(seed: int, keys: np.ndarray, lo: float, hi: float) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.zeros(keys.shape[0])
    check(lib().cf_counter_uniform(int(seed), keys.ctypes.data_as(C.POINTER(C.c_int64)), keys.shape[0], lo, hi,
                                   out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


# ------------------------------------------------------------------ text formats
def _text_arg(text) -> bytes:
    return text.encode() if isinstance(text, str) else bytes(text)


def _format(fn, *args) -> str:
    n = C.c_int64(0)
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.raw[:n.value].decode()


def _table(t: "_abi.cf_table") -> PiecewiseLinear:
    return PiecewiseLinear([t.x[i] for i in range(t.n)], [t.y[i] for i in range(t.n)])


def _mesh_from_handle(h) -> Mesh:
    try:
        d = _abi.cf_mesh_desc()
        check(lib().cf_mesh_view(h, C.byref(d)))
        N, E, F = d.n_nodes, d.n_elems, d.n_facets
        arr = lambda ptr, n, dt: np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True) if n else np.zeros(0, dt)
        return Mesh(arr(d.coords, 3 * N, np.float64).reshape(-1, 3), arr(d.tets, 4 * E, np.int32).reshape(-1, 4),
                    arr(d.region, E, np.int32), arr(d.facets, 3 * F, np.int32).reshape(-1, 3),
                    arr(d.facet_tag, F, np.int32), [d.tags[i].decode() for i in range(d.n_tags)],
                    [(d.contacts[2 * i], d.contacts[2 * i + 1]) for i in range(d.n_contacts)])
    finally:
        lib().cf_mesh_free(h)


def parse_mesh(text) -> Mesh:
    """parse_mesh (mesh.hpp:256-325): 'femesh 1' text -> a finalized Mesh (oriented tets).
    Raises ParseError (line-numbered) / ValidationError like the reference."""
    b = _text_arg(text)
    h = C.c_void_p()
    check(lib().cf_mesh_parse(b, len(b), C.byref(h)))
    return _mesh_from_handle(h)


def write_mesh(m: Mesh) -> str:
    """write_mesh (mesh.hpp:327-343)."""
    keep = _Keep()
    return _format(lib().cf_mesh_format, C.byref(mesh_desc(m, keep)))


MESH_BINARY_MAGIC = b"CFMESHB1"


def parse_mesh_binary(data: bytes) -> Mesh:
    """The binary fast path ("CFMESHB1"): same validation / orientation as parse_mesh."""
    b = bytes(data)
    h = C.c_void_p()
    check(lib().cf_mesh_parse_binary(b, len(b), C.byref(h)))
    return _mesh_from_handle(h)


def write_mesh_binary(m: Mesh) -> bytes:
    keep = _Keep()
    d = mesh_desc(m, keep)
    n = C.c_int64(0)
    check(lib().cf_mesh_format_binary(C.byref(d), None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(1, n.value))
    check(lib().cf_mesh_format_binary(C.byref(d), buf, n.value, C.byref(n)))
    return buf.raw[:n.value]


def read_mesh(path: str) -> Mesh:
    """A mesh file: the reference's femesh text, or this repo's binary fast path (by magic)."""
    with open(path, "rb") as f:
        data = f.read()
    return parse_mesh_binary(data) if data[:8] == MESH_BINARY_MAGIC else parse_mesh(data)


def parse_config(text) -> SimulationSetup:
    """parse_config (material.hpp:186-345) -> SimulationSetup (materials indexed by region,
    boundary conditions by tag, interface coefficients, solver)."""
    b = _text_arg(text)
    h = C.c_void_p()
    check(lib().cf_config_parse(b, len(b), C.byref(h)))
    try:
        d = _abi.cf_setup_desc()
        check(lib().cf_config_view(h, C.byref(d)))
        mats = [MaterialTable(m.rho, _table(m.c), _table(m.k), m.latent_heat, m.solidus, m.liquidus,
                              m.initial_temperature) for m in (d.materials[i] for i in range(d.n_materials))]
        bcs = {}
        for i in range(d.n_bcs):
            b_ = d.bcs[i]
            bcs[b_.tag.decode()] = BoundaryCondition("fixed" if b_.kind == _abi.CF_BC_FIXED else "flux",
                                                     _table(b_.fixed_T), b_.q, b_.h, b_.t_inf)
        cos = [InterfaceCoeff(c.tag_a.decode(), c.tag_b.decode(),
                              "temperature" if c.var == _abi.CF_VAR_TEMPERATURE else "time", _table(c.h))
               for c in (d.coeffs[i] for i in range(d.n_coeffs))]
        return SimulationSetup(materials=mats, boundary_conditions=bcs, interface_coeffs=cos,
                               solver=SolverConfig(d.dt_safety, d.t_end, int(d.output_every)))
    finally:
        lib().cf_config_free(h)


def load_partmap(text, element_count: int) -> Tuple[np.ndarray, int]:
    """load_partmap (partition.hpp:424-445) -> (part_of_element, part_count)."""
    b = _text_arg(text)
    out = np.zeros(max(1, element_count), dtype=np.int32)
    count = C.c_int32(0)
    check(lib().cf_partmap_parse(b, len(b), int(element_count), out.ctypes.data_as(_abi._ip), C.byref(count)))
    return out[:element_count], int(count.value)


def write_partmap(parts: np.ndarray) -> str:
    """write_partmap (partition.hpp:447-449)."""
    p = np.ascontiguousarray(parts, dtype=np.int32)
    return _format(lib().cf_partmap_format, p.ctypes.data_as(_abi._ip), len(p))


# ------------------------------------------------------------------ tile autotuner
@dataclass
class TuneReport:
    """TuneReport (blocked.hpp:558-563): candidates (elements per tile), best-of-2 device
    seconds of trial_steps per candidate, the chosen one, tune overhead fraction."""
    candidates: List[int]
    seconds: List[float]
    chosen: int
    overhead_fraction: float = 0.0


def choose_tile_elems(candidates: Sequence[int], seconds: Sequence[float]) -> int:
    """choose_block_count (blocked.hpp:566-575): argmin, the first candidate wins ties."""
    c = np.ascontiguousarray(candidates, dtype=np.int32)
    t = np.ascontiguousarray(seconds, dtype=np.float64)
    out = C.c_int32(0)
    check(lib().cf_choose_tile_elems(c.ctypes.data_as(_abi._ip), t.ctypes.data_as(_abi._dp),
                                     len(c) if len(c) == len(t) else -1, C.byref(out)))
    return int(out.value)


def default_tile_candidates(element_count: int) -> List[int]:
    """default_block_candidates (blocked.hpp:578-583) recast: 6*2^k tets per tile (cell boxes
    of structured meshes in Morton order), at least one tile per SM."""
    out = np.zeros(16, dtype=np.int32)
    n = C.c_int32(0)
    check(lib().cf_default_tile_candidates(int(element_count), out.ctypes.data_as(_abi._ip), 16, C.byref(n)))
    return [int(v) for v in out[:n.value]]


def autotune_tiles(m: Mesh, setup: SimulationSetup, opts: Optional[SolveOptions] = None,
                   candidates: Optional[Sequence[int]] = None, trial_steps: int = 10,
                   projected_total_steps: float = 0.0) -> TuneReport:
    """autotune_block_count (blocked.hpp:587-623) recast for the B200: builds a plan per
    candidate tile size and times trial_steps (best of 2, device time) from the initial field."""
    keep = _Keep()
    md, sd = mesh_desc(m, keep), setup_desc(setup, keep)
    ro = run_opts(opts or SolveOptions(), keep)
    cand = np.ascontiguousarray(candidates if candidates is not None else default_tile_candidates(m.element_count()),
                                dtype=np.int32)
    secs = np.zeros(max(1, len(cand)))
    rep = _abi.cf_tune_report()
    check(lib().cf_autotune_tiles(C.byref(md), C.byref(sd), C.byref(ro), cand.ctypes.data_as(_abi._ip), len(cand),
                                  int(trial_steps), float(projected_total_steps), secs.ctypes.data_as(_abi._dp),
                                  C.byref(rep)))
    return TuneReport([int(c) for c in cand], [float(x) for x in secs[:len(cand)]], int(rep.chosen),
                      float(rep.overhead_fraction))

