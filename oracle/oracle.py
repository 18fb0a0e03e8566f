"""ctypes access to the CPU checkers — TEST INFRASTRUCTURE ONLY.

  liboracle.so            the plain-C restatement (castfem_oracle.c)
  _ref/libcastfem_ref.so  the unmodified reference headers behind ref_driver.cpp

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may use this module. Descriptor structs come from the
product's ABI mirror (they are the boundary definition, not product logic).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_1005_3158_b200 import _abi
from paper_1005_3158_b200.castfem import Mesh, SimulationSetup, _Keep, mesh_desc, setup_desc

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcastfem_ref.so")
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class or_result(C.Structure):
    _fields_ = [("time", C.c_double), ("dt", C.c_double), ("static_dt", C.c_double), ("loop_seconds", C.c_double),
                ("steps", C.c_int64), ("clamp_steps", C.c_int64), ("n_series", C.c_int64),
                ("dynamic_dt", C.c_int32)]


_o = None
_r = None


def oracle_lib():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        L.or_solve.restype = C.c_int
        L.or_solve.argtypes = [C.POINTER(_abi.cf_mesh_desc), C.POINTER(_abi.cf_setup_desc), _ip, C.c_int32, _ip,
                               C.c_int32, C.c_int64, _dp, _dp, _dp, C.c_int64, C.POINTER(or_result)]
        L.or_last_error.restype = C.c_char_p
        L.or_lambda_max.restype = C.c_int
        L.or_lambda_max.argtypes = [C.POINTER(_abi.cf_mesh_desc), C.POINTER(_abi.cf_setup_desc), C.c_int,
                                    C.c_uint64, _dp, _dp]
        L.or_pair_sister_facets.argtypes = [C.POINTER(_abi.cf_mesh_desc), _ip, C.c_int64, C.POINTER(C.c_int64)]
        L.or_tet_geometry.argtypes = [_dp, _dp]
        L.or_enthalpy.restype = C.c_double
        L.or_enthalpy.argtypes = [C.POINTER(_abi.cf_material), C.c_double]
        L.or_apparent_heat_capacity.restype = C.c_double
        L.or_apparent_heat_capacity.argtypes = [_dp, _dp, _dp, C.POINTER(_abi.cf_material)]
        L.or_assemble_part.restype = C.c_int
        L.or_assemble_part.argtypes = [C.POINTER(_abi.cf_mesh_desc), C.POINTER(_abi.cf_setup_desc), C.c_char_p, _dp,
                                       _dp, C.c_double, _dp, _dp]
        L.or_generate_fixture.restype = C.c_int
        L.or_generate_fixture.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_uint64, _ip,
                                          C.POINTER(_abi.cf_fixture)]
        L.or_counter_uniform_array.restype = None
        L.or_counter_uniform_array.argtypes = [C.c_uint64, C.POINTER(C.c_int64), C.c_int64, C.c_double, C.c_double,
                                               _dp]
        L.or_element_accumulate.restype = None
        L.or_element_accumulate.argtypes = [_dp, C.POINTER(_abi.cf_material), _dp, _dp, _dp, _dp]
        _o = L
    return _o


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _r
    if _r is None:
        if not os.path.exists(REF_SO):
            raise ImportError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_solve.restype = C.c_int
        L.ref_solve.argtypes = [C.POINTER(_abi.cf_mesh_desc), C.POINTER(_abi.cf_setup_desc), C.c_int32, C.c_int64,
                                _dp, _dp, _dp, _ip, _dp, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_bench_create.restype = C.c_void_p
        L.ref_bench_create.argtypes = [C.POINTER(_abi.cf_mesh_desc), C.POINTER(_abi.cf_setup_desc)]
        L.ref_bench_steps.restype = C.c_double
        L.ref_bench_steps.argtypes = [C.c_void_p, C.c_int64]
        L.ref_bench_get_T.argtypes = [C.c_void_p, _dp]
        L.ref_bench_destroy.argtypes = [C.c_void_p]
        L.ref_pair_sister_facets.argtypes = [C.POINTER(_abi.cf_mesh_desc), _ip, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_finalize.argtypes = [C.POINTER(_abi.cf_mesh_desc), _ip, _ip]
        L.ref_rcm_permutation.argtypes = [C.POINTER(_abi.cf_mesh_desc), C.c_int32, _ip]
        L.ref_bandwidth.argtypes = [C.POINTER(_abi.cf_mesh_desc), _ip, C.POINTER(C.c_int64)]
        L.ref_tet_geometry.argtypes = [_dp, _dp]
        L.ref_enthalpy.restype = C.c_double
        L.ref_enthalpy.argtypes = [C.POINTER(_abi.cf_material), C.c_double]
        L.ref_apparent_heat_capacity.restype = C.c_double
        L.ref_apparent_heat_capacity.argtypes = [_dp, _dp, _dp, C.POINTER(_abi.cf_material)]
        for f in (L.ref_mesh_roundtrip, L.ref_config_dump):
            f.restype = C.c_int
            f.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_partition.restype = C.c_int
        L.ref_partition.argtypes = [C.POINTER(_abi.cf_mesh_desc), C.c_int32, C.c_double, C.c_int32, _ip]
        L.ref_partition_metrics.restype = C.c_int
        L.ref_partition_metrics.argtypes = [C.POINTER(_abi.cf_mesh_desc), _ip, C.c_int32, C.POINTER(C.c_int64), _dp,
                                            _ip, C.POINTER(C.c_int64)]
        L.ref_load_partmap.restype = C.c_int
        L.ref_load_partmap.argtypes = [C.c_char_p, C.c_int64, C.c_int32, _ip, C.POINTER(C.c_int32)]
        _r = L
    return _r


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class OracleResult:
    T: np.ndarray
    H: np.ndarray
    time: float
    dt: float
    steps: int
    clamp_steps: int
    loop_seconds: float
    static_dt: float
    series: np.ndarray


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def solve(mesh: Mesh, setup: SimulationSetup, max_steps: int, blocks: Optional[np.ndarray] = None,
          parts: Optional[np.ndarray] = None) -> OracleResult:
    """The C restatement: blocks = element->block map (BlockPlan semantics), parts = element->worker."""
    keep = _Keep()
    md, sd = mesh_desc(mesh, keep), setup_desc(setup, keep)
    N = mesh.node_count()
    T = np.zeros(N)
    H = np.zeros(N)
    ser = np.zeros(3 * 4096)
    res = or_result()
    b = np.ascontiguousarray(blocks, dtype=np.int32) if blocks is not None else None
    pp = np.ascontiguousarray(parts, dtype=np.int32) if parts is not None else None
    nb = int(b.max()) + 1 if b is not None and len(b) else 1
    npart = int(pp.max()) + 1 if pp is not None and len(pp) else 1
    st = oracle_lib().or_solve(C.byref(md), C.byref(sd), _p(b, C.c_int32), nb, _p(pp, C.c_int32), npart,
                               int(max_steps), _p(T), _p(H), _p(ser), 4096, C.byref(res))
    if st:
        raise OracleError(st, oracle_lib().or_last_error().decode())
    ns = min(res.n_series, 4096)
    return OracleResult(T, H, res.time, res.dt, res.steps, res.clamp_steps, res.loop_seconds, res.static_dt,
                        ser[:3 * ns].reshape(-1, 3))


def ref_solve(mesh: Mesh, setup: SimulationSetup, max_steps: int, blocks: int = 1):
    """The reference itself (oracle/_ref). Returns (OracleResult, block_map)."""
    keep = _Keep()
    md, sd = mesh_desc(mesh, keep), setup_desc(setup, keep)
    N = mesh.node_count()
    T = np.zeros(N)
    H = np.zeros(N)
    stats = np.zeros(8)
    bm = np.zeros(mesh.element_count(), np.int32)
    ser = np.zeros(3 * 4096)
    ns = C.c_int64()
    st = ref_lib().ref_solve(C.byref(md), C.byref(sd), int(blocks), int(max_steps), _p(T), _p(H), _p(stats),
                             _p(bm, C.c_int32), _p(ser), 4096, C.byref(ns))
    if st:
        raise OracleError(st, ref_lib().ref_last_error().decode())
    k = min(ns.value, 4096)
    r = OracleResult(T, H, stats[0], stats[1], int(stats[2]), int(stats[3]), stats[4], stats[5],
                     ser[:3 * k].reshape(-1, 3))
    return r, bm


def lambda_max(mesh: Mesh, setup: SimulationSetup, iterations: int = 500, seed: int = 1234):
    keep = _Keep()
    md, sd = mesh_desc(mesh, keep), setup_desc(setup, keep)
    lam, e13 = C.c_double(), C.c_double()
    st = oracle_lib().or_lambda_max(C.byref(md), C.byref(sd), iterations, seed, C.byref(lam), C.byref(e13))
    if st:
        raise OracleError(st, oracle_lib().or_last_error().decode())
    return lam.value, e13.value


class RefBench:
    """Reference blocked_step loop on one host core (bench --impl reference)."""

    def __init__(self, mesh: Mesh, setup: SimulationSetup):
        self._keep = _Keep()
        md, sd = mesh_desc(mesh, self._keep), setup_desc(setup, self._keep)
        self.h = ref_lib().ref_bench_create(C.byref(md), C.byref(sd))
        if not self.h:
            raise OracleError(-1, ref_lib().ref_last_error().decode())
        self.N = mesh.node_count()

    def steps(self, n: int) -> float:
        secs = ref_lib().ref_bench_steps(self.h, int(n))
        if secs < 0:
            raise OracleError(int(-secs), ref_lib().ref_last_error().decode())
        return secs

    def T(self) -> np.ndarray:
        T = np.zeros(self.N)
        ref_lib().ref_bench_get_T(self.h, _p(T))
        return T

    def close(self):
        if self.h:
            ref_lib().ref_bench_destroy(self.h)
            self.h = None


def assemble_part(mesh: Mesh, setup: SimulationSetup, elem_mask: np.ndarray, T: np.ndarray, T_old: np.ndarray,
                  time: float):
    """Per-node (c, r) of one worker's elements (ascending element order, its facets after)."""
    keep = _Keep()
    md, sd = mesh_desc(mesh, keep), setup_desc(setup, keep)
    N = mesh.node_count()
    c = np.zeros(N)
    r = np.zeros(N)
    mask = np.ascontiguousarray(elem_mask, dtype=np.int8)
    T = np.ascontiguousarray(T, dtype=np.float64)
    T_old = np.ascontiguousarray(T_old, dtype=np.float64)
    st = oracle_lib().or_assemble_part(C.byref(md), C.byref(sd), mask.ctypes.data_as(C.c_char_p), _p(T), _p(T_old),
                                       time, _p(c), _p(r))
    if st:
        raise OracleError(st, oracle_lib().or_last_error().decode())
    return c, r


# ---------------------------------------------------------------- text formats (reference parsers)
def _ref_text(fn, text: bytes):
    n = C.c_int64(0)
    st = fn(text, len(text), None, 0, C.byref(n))
    if st:
        return st, ref_lib().ref_last_error().decode()
    buf = C.create_string_buffer(n.value + 1)
    fn(text, len(text), buf, n.value + 1, C.byref(n))
    return 0, buf.raw[:n.value].decode()


def ref_mesh_roundtrip(text: bytes):
    """(status, text): the reference's parse_mesh -> write_mesh, or (status, error message)."""
    return _ref_text(ref_lib().ref_mesh_roundtrip, text)


def ref_config_dump(text: bytes):
    """(status, canonical dump of the reference's parse_config), or (status, error message)."""
    return _ref_text(ref_lib().ref_config_dump, text)


def ref_load_partmap(text: bytes, n_elems: int):
    out = np.zeros(max(1, n_elems), dtype=np.int32)
    count = C.c_int32(0)
    st = ref_lib().ref_load_partmap(text, len(text), int(n_elems), _p(out, C.c_int32), C.byref(count))
    if st:
        return st, ref_lib().ref_last_error().decode()
    return 0, (out[:n_elems], int(count.value))



# ---------------------------------------------------------------- fixtures (oracle/fixture.c)
REF_BENCH = os.path.join(HERE, "_ref", "ref_bench")


def generate_fixture(kind: str, n: int, radius: float = 0.35, jitter: float = 0.0, seed: int = 0,
                     perm_seed: int = 0, window=None) -> dict:
    """The oracle's restatement of the synthetic workload generator (arrays as a dict)."""
    k = {"cube": 0, "casting": 1}[kind]
    w = np.ascontiguousarray(np.asarray(window, dtype=np.int32).reshape(6)) if window is not None else None
    fx = _abi.cf_fixture()
    wp = _p(w, C.c_int32)
    st = oracle_lib().or_generate_fixture(k, n, radius, jitter, seed, perm_seed, wp, C.byref(fx))
    if st:
        raise OracleError(st, "bad fixture arguments")
    out = {"nodes": np.zeros((fx.n_nodes, 3)), "tets": np.zeros((fx.n_elems, 4), np.int32),
           "region": np.zeros(fx.n_elems, np.int32), "facets": np.zeros((fx.n_facets, 3), np.int32),
           "facet_tag": np.zeros(fx.n_facets, np.int32), "node_grid": np.zeros(fx.n_nodes, np.int32)}
    fx.coords = _p(out["nodes"])
    fx.tets = _p(out["tets"], C.c_int32)
    fx.region = _p(out["region"], C.c_int32)
    fx.facets = _p(out["facets"], C.c_int32)
    fx.facet_tag = _p(out["facet_tag"], C.c_int32)
    fx.node_grid = _p(out["node_grid"], C.c_int32)
    st = oracle_lib().or_generate_fixture(k, n, radius, jitter, seed, perm_seed, wp, C.byref(fx))
    if st:
        raise OracleError(st, "fixture generation failed")
    return out


def counter_uniform(seed: int, keys: np.ndarray, lo: float, hi: float) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    out = np.zeros(keys.shape[0])
    oracle_lib().or_counter_uniform_array(seed, keys.ctypes.data_as(C.POINTER(C.c_int64)), keys.shape[0], lo, hi,
                                          _p(out))
    return out


def ref_bench(workload: str, steps: int = 10, warmup: int = 1, window=None, blocks: int = 1, autotune=None,
              describe: bool = False, dump_T: Optional[str] = None, timeout: float = 3600) -> dict:
    """Runs oracle/_ref/ref_bench (the reference's own blocked_step loop in its own process)."""
    import json
    import subprocess
    if not os.path.exists(REF_BENCH):
        raise ImportError(f"{REF_BENCH} missing: run `make -C oracle` where /root/reference exists")
    cmd = [REF_BENCH, "--workload", workload, "--steps", str(steps), "--warmup", str(warmup), "--blocks", str(blocks)]
    if window is not None:
        w = list(window)
        cmd += ["--window", f"{w[0]}:{w[1]},{w[2]}:{w[3]},{w[4]}:{w[5]}"]
    if autotune:
        cmd += ["--autotune", ",".join(str(c) for c in autotune)]
    if describe:
        cmd.append("--describe")
    if dump_T:
        cmd += ["--dump-T", dump_T]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
    if out.returncode != 0:
        raise OracleError(out.returncode, out.stderr.strip())
    return json.loads(out.stdout.strip().splitlines()[-1])
