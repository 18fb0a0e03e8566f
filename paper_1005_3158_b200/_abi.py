"""ctypes mirror of include/castfem_b200.h (the C-ABI boundary).

Loads the in-tree ``libcastfem_b200.so``. There is no fallback: if the
library is missing the import fails loudly (build it with
``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CF_LIB_PATH") or os.path.join(_HERE, "libcastfem_b200.so")

CF_OK, CF_PARSE, CF_VALIDATION, CF_CONFIG, CF_PROTOCOL, CF_DEGENERATE, CF_CUDA, CF_NCCL, CF_INVALID_ARG = range(9)
CF_BC_FLUX, CF_BC_FIXED = 0, 1
CF_VAR_TIME, CF_VAR_TEMPERATURE = 0, 1
CF_MODE_ATOMIC, CF_MODE_DETERMINISTIC = 0, 1
CF_NODE_ORDER_GIVEN, CF_NODE_ORDER_RCM, CF_NODE_ORDER_TILE = 0, 1, 2
CF_ELEM_ORDER_GIVEN, CF_ELEM_ORDER_MORTON, CF_ELEM_ORDER_MIN_NODE = 0, 1, 2
CF_GEOM_STORED, CF_GEOM_COORDS = 0, 1
CF_PARTITION_RCB, CF_PARTITION_GIVEN, CF_PARTITION_GRAPH = 0, 1, 2

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class cf_table(C.Structure):
    _fields_ = [("n", C.c_int32), ("x", _dp), ("y", _dp)]


class cf_material(C.Structure):
    _fields_ = [("rho", C.c_double), ("c", cf_table), ("k", cf_table), ("latent_heat", C.c_double),
                ("solidus", C.c_double), ("liquidus", C.c_double), ("initial_temperature", C.c_double)]


class cf_boundary_condition(C.Structure):
    _fields_ = [("tag", C.c_char_p), ("kind", C.c_int32), ("fixed_T", cf_table), ("q", C.c_double),
                ("h", C.c_double), ("t_inf", C.c_double)]


class cf_interface_coeff(C.Structure):
    _fields_ = [("tag_a", C.c_char_p), ("tag_b", C.c_char_p), ("var", C.c_int32), ("h", cf_table)]


class cf_mesh_desc(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("coords", _dp), ("n_elems", C.c_int32), ("tets", _ip),
                ("region", _ip), ("n_facets", C.c_int32), ("facets", _ip), ("facet_tag", _ip),
                ("n_tags", C.c_int32), ("tags", C.POINTER(C.c_char_p)), ("n_contacts", C.c_int32),
                ("contacts", _ip)]


class cf_setup_desc(C.Structure):
    _fields_ = [("n_materials", C.c_int32), ("materials", C.POINTER(cf_material)), ("n_bcs", C.c_int32),
                ("bcs", C.POINTER(cf_boundary_condition)), ("n_coeffs", C.c_int32),
                ("coeffs", C.POINTER(cf_interface_coeff)), ("dt_safety", C.c_double), ("t_end", C.c_double),
                ("output_every", C.c_int64), ("initial_T", _dp)]


class cf_run_opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("mode", C.c_int32), ("node_order", C.c_int32), ("elem_order", C.c_int32),
                ("tile_elems", C.c_int32), ("tile_of_element", _ip), ("n_tiles_given", C.c_int32),
                ("fast_math", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32),
                ("local_ranks", C.c_int32), ("partition", C.c_int32), ("part_of_element", _ip),
                ("comm", C.c_void_p), ("geometry", C.c_int32)]


class cf_stats(C.Structure):
    _fields_ = [("time", C.c_double), ("dt", C.c_double), ("step_index", C.c_int64), ("clamp_steps", C.c_int64),
                ("loop_seconds", C.c_double), ("static_dt", C.c_double), ("dynamic_dt", C.c_int32),
                ("n_tiles", C.c_int32), ("n_elems_local", C.c_int64), ("n_nodes_local", C.c_int64),
                ("total_slots", C.c_int64), ("n_shared_nodes", C.c_int64), ("n_ghost_nodes", C.c_int64),
                ("device_bytes", C.c_int64), ("bytes_per_step", C.c_int64), ("launches_per_step", C.c_int64),
                ("tile_bytes_per_launch", C.c_int64), ("update_bytes_per_step", C.c_int64),
                ("n_nodes_global", C.c_int64), ("n_elems_global", C.c_int64), ("device_setup", C.c_int32)]


class cf_tune_report(C.Structure):
    _fields_ = [("n_candidates", C.c_int32), ("chosen", C.c_int32), ("overhead_fraction", C.c_double)]


class cf_fixture(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_elems", C.c_int32), ("n_facets", C.c_int32), ("coords", _dp),
                ("tets", _ip), ("region", _ip), ("facets", _ip), ("facet_tag", _ip), ("node_grid", _ip)]


class cf_fixture_spec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("radius", C.c_double), ("jitter", C.c_double),
                ("seed", C.c_uint64), ("perm_seed", C.c_uint64), ("t0_noise", C.c_double), ("noise_seed", C.c_uint64),
                ("rcm", C.c_int32)]


CF_REDUCE_MIN, CF_REDUCE_MAX = 0, 1
SENDRECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, _ip, C.POINTER(_dp), C.POINTER(C.c_int64),
                          C.POINTER(_dp), C.POINTER(C.c_int64))
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, _dp, C.c_int64, C.c_int32)


class cf_host_transport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("sendrecv", SENDRECV_FN), ("allreduce", ALLREDUCE_FN)]


# (name, restype, argtypes) — every symbol declared in include/castfem_b200.h
SIGNATURES = [
    ("cf_abi_version", C.c_int, []),
    ("cf_last_error", C.c_int, [C.c_char_p, C.c_size_t]),
    ("cf_plan_create", C.c_int, [C.POINTER(cf_mesh_desc), C.POINTER(cf_setup_desc), C.POINTER(cf_run_opts),
                                 C.POINTER(C.c_void_p)]),
    ("cf_plan_destroy", C.c_int, [C.c_void_p]),
    ("cf_set_temperature", C.c_int, [C.c_void_p, _dp]),
    ("cf_set_dt_safety", C.c_int, [C.c_void_p, C.c_double]),
    ("cf_step", C.c_int, [C.c_void_p, C.c_int64, C.c_double]),
    ("cf_solve", C.c_int, [C.c_void_p, C.c_int64, _dp, C.c_int64, C.POINTER(C.c_int64)]),
    ("cf_get_fields", C.c_int, [C.c_void_p, _dp, _dp]),
    ("cf_get_stats", C.c_int, [C.c_void_p, C.POINTER(cf_stats)]),
    ("cf_device_temperature", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(_dp), C.POINTER(C.c_int64)]),
    ("cf_enable_graph", C.c_int, [C.c_void_p, C.c_int64]),
    ("cf_time_phases", C.c_int, [C.c_void_p, C.c_int64, _dp]),
    ("cf_estimate_lambda_max", C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, _dp, _dp]),
    ("cf_comm_unique_id", C.c_int, [C.c_char_p]),
    ("cf_comm_create", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_void_p)]),
    ("cf_comm_create_host", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(cf_host_transport),
                                      C.POINTER(C.c_void_p)]),
    ("cf_comm_create_peer", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(cf_host_transport),
                                      C.POINTER(C.c_void_p)]),
    ("cf_comm_destroy", C.c_int, [C.c_void_p]),
    ("cf_rcm_permutation", C.c_int, [C.POINTER(cf_mesh_desc), C.c_int32, _ip]),
    ("cf_rcm_permutation_device", C.c_int, [C.POINTER(cf_mesh_desc), C.c_int32, C.c_int32, _ip]),
    ("cf_bandwidth", C.c_int, [C.POINTER(cf_mesh_desc), _ip, C.POINTER(C.c_int64)]),
    ("cf_finalize_mesh", C.c_int, [C.POINTER(cf_mesh_desc), _ip, _ip]),
    ("cf_pair_sister_facets", C.c_int, [C.POINTER(cf_mesh_desc), _ip, C.c_int64, C.POINTER(C.c_int64)]),
    ("cf_partition_rcb", C.c_int, [C.POINTER(cf_mesh_desc), C.c_int32, _ip]),
    ("cf_partition_graph", C.c_int, [C.POINTER(cf_mesh_desc), C.c_int32, C.c_double, C.c_int32, _ip]),
    ("cf_partition_metrics", C.c_int, [C.POINTER(cf_mesh_desc), _ip, C.c_int32, C.POINTER(C.c_int64), _dp, _ip,
                                       C.POINTER(C.c_int64)]),
    ("cf_tile_map", C.c_int, [C.POINTER(cf_mesh_desc), C.POINTER(cf_setup_desc), C.POINTER(cf_run_opts), _ip,
                              _ip]),
    ("cf_plan_create_fixture", C.c_int, [C.POINTER(cf_fixture_spec), C.POINTER(cf_setup_desc),
                                         C.POINTER(cf_run_opts), C.POINTER(C.c_void_p)]),
    ("cf_plan_digest_device", C.c_int, [C.POINTER(cf_mesh_desc), C.POINTER(cf_setup_desc), C.POINTER(cf_run_opts),
                                        C.c_int32, C.POINTER(C.c_uint64)]),
    ("cf_partition_rcb_device", C.c_int, [C.POINTER(cf_mesh_desc), C.c_int32, _ip]),
    ("cf_plan_digest", C.c_int, [C.POINTER(cf_mesh_desc), C.POINTER(cf_setup_desc), C.POINTER(cf_run_opts),
                                 C.c_int32, C.POINTER(C.c_uint64)]),
    ("cf_exchange_plan", C.c_int, [C.POINTER(cf_mesh_desc), C.POINTER(cf_setup_desc), C.POINTER(cf_run_opts), _ip,
                                   _ip, C.POINTER(C.c_int64), _ip, _ip, _ip]),
    ("cf_generate_fixture", C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                                      C.POINTER(cf_fixture)]),
    ("cf_counter_uniform", C.c_int, [C.c_uint64, C.POINTER(C.c_int64), C.c_int64, C.c_double, C.c_double, _dp]),
    ("cf_autotune_tiles", C.c_int, [C.POINTER(cf_mesh_desc), C.POINTER(cf_setup_desc), C.POINTER(cf_run_opts),
                                    _ip, C.c_int32, C.c_int32, C.c_double, _dp, C.POINTER(cf_tune_report)]),
    ("cf_choose_tile_elems", C.c_int, [_ip, _dp, C.c_int32, C.POINTER(C.c_int32)]),
    ("cf_default_tile_candidates", C.c_int, [C.c_int64, _ip, C.c_int32, C.POINTER(C.c_int32)]),
    ("cf_mesh_parse", C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_void_p)]),
    ("cf_mesh_view", C.c_int, [C.c_void_p, C.POINTER(cf_mesh_desc)]),
    ("cf_mesh_free", None, [C.c_void_p]),
    ("cf_mesh_format", C.c_int, [C.POINTER(cf_mesh_desc), C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]),
    ("cf_mesh_parse_binary", C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)]),
    ("cf_mesh_format_binary", C.c_int, [C.POINTER(cf_mesh_desc), C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    ("cf_config_parse", C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_void_p)]),
    ("cf_config_view", C.c_int, [C.c_void_p, C.POINTER(cf_setup_desc)]),
    ("cf_config_free", None, [C.c_void_p]),
    ("cf_partmap_parse", C.c_int, [C.c_char_p, C.c_int64, C.c_int32, _ip, C.POINTER(C.c_int32)]),
    ("cf_partmap_format", C.c_int, [_ip, C.c_int32, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]),
]

_lib = None


def lib() -> C.CDLL:
    """The product library; raises if it was not built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with __graft_entry__.build() — there is no CPU fallback")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    buf = C.create_string_buffer(1024)
    lib().cf_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")
