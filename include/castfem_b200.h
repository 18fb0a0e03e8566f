/*
 * castfem_b200.h — C-ABI drop-in boundary for the explicit element-by-element
 * FE step of the `castfem` reference solver (arXiv 1005.3158), B200-native.
 *
 * The reference exposes no FFI: its boundary is the header-only C++ API in
 * /root/reference/proj/include/castfem/. Every entry point below names the
 * reference interface it replaces (file:line, paths relative to
 * proj/include/castfem/). Conventions:
 *   - plain pointers + sizes, no C++ or torch types; int32 ids, int64 counts;
 *   - nothing the caller passes is retained after a call returns;
 *   - every function returns a status (CF_OK = 0); the message of the last
 *     failure on the calling thread is available through cf_last_error();
 *   - reference exceptions map to status codes (errors.hpp:8-31,
 *     geometry.hpp:43-46); device-side failures (c_diag <= 0) report
 *     CF_VALIDATION with the offending global node id, as
 *     explicit_update (fem.hpp:107-114) throws validation_error.
 *
 * A plan is not thread-safe; distinct plans are independent.
 */
#ifndef CASTFEM_B200_H
#define CASTFEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CF_ABI_VERSION 2

/* status codes — errors.hpp:8-31 (+ degenerate_element_error geometry.hpp:43-46) */
enum {
    CF_OK = 0,
    CF_PARSE = 1,        /* parse_error        errors.hpp:8-16  */
    CF_VALIDATION = 2,   /* validation_error   errors.hpp:18-21 */
    CF_CONFIG = 3,       /* config_error       errors.hpp:23-26 */
    CF_PROTOCOL = 4,     /* protocol_error     errors.hpp:28-31 */
    CF_DEGENERATE = 5,   /* degenerate_element_error geometry.hpp:43-46 */
    CF_CUDA = 6,         /* CUDA runtime failure (no reference analogue) */
    CF_NCCL = 7,         /* NCCL failure (no reference analogue) */
    CF_INVALID_ARG = 8   /* null pointer / bad size at the boundary */
};

/* ---------------------------------------------------------------------------
 * Problem description (copied at cf_plan_create; mirrors the reference types)
 * ------------------------------------------------------------------------- */

/* PiecewiseLinear (material.hpp:21-47): n == 1 is a constant (never clamps);
 * n >= 2 clamps to the covered range; n == 0 is "unset". */
typedef struct cf_table {
    int32_t n;
    const double* x;
    const double* y;
} cf_table;

/* MaterialTable (material.hpp:53-124); one per region id. */
typedef struct cf_material {
    double rho;
    cf_table c;          /* c(T)  J/kgK */
    cf_table k;          /* k(T)  W/mK  */
    double latent_heat;  /* J/kg; 0 = no phase change */
    double solidus;
    double liquidus;
    double initial_temperature;
} cf_material;

/* BoundaryCondition (material.hpp:126-141), keyed by facet tag name. */
enum { CF_BC_FLUX = 0, CF_BC_FIXED = 1 };
typedef struct cf_boundary_condition {
    const char* tag;
    int32_t kind;        /* CF_BC_FLUX | CF_BC_FIXED */
    cf_table fixed_T;    /* of time, for CF_BC_FIXED (fixed_fn is not expressible in C) */
    double q;            /* imposed flux W/m^2, positive = heat leaving */
    double h;            /* convective coefficient W/m^2K */
    double t_inf;        /* ambient K */
} cf_boundary_condition;

/* InterfaceCoeff (material.hpp:145-153). */
enum { CF_VAR_TIME = 0, CF_VAR_TEMPERATURE = 1 };
typedef struct cf_interface_coeff {
    const char* tag_a;
    const char* tag_b;
    int32_t var;         /* CF_VAR_TIME | CF_VAR_TEMPERATURE */
    cf_table h;
} cf_interface_coeff;

/* Mesh (mesh.hpp:45-80): nodes, tets (+region), tagged boundary facets,
 * contact declarations (pairs of tag ids). Ids are 0-based. */
typedef struct cf_mesh_desc {
    int32_t n_nodes;
    const double* coords;      /* [3*n_nodes] x,y,z */
    int32_t n_elems;
    const int32_t* tets;       /* [4*n_elems] */
    const int32_t* region;     /* [n_elems] */
    int32_t n_facets;
    const int32_t* facets;     /* [3*n_facets] */
    const int32_t* facet_tag;  /* [n_facets] index into tags */
    int32_t n_tags;
    const char* const* tags;   /* [n_tags] */
    int32_t n_contacts;
    const int32_t* contacts;   /* [2*n_contacts] (tag_a = cast side, tag_b) */
} cf_mesh_desc;

/* SimulationSetup (material.hpp:162-184) + SolverConfig (:155-160). */
typedef struct cf_setup_desc {
    int32_t n_materials;
    const cf_material* materials;     /* indexed by region id */
    int32_t n_bcs;
    const cf_boundary_condition* bcs;
    int32_t n_coeffs;
    const cf_interface_coeff* coeffs;
    double dt_safety;                 /* (0, 1] */
    double t_end;
    int64_t output_every;             /* 0 disables the series */
    const double* initial_T;          /* optional [n_nodes]; replaces initial_override (:167-168) */
} cf_setup_desc;

/* ---------------------------------------------------------------------------
 * Run options (the B200 recast of SolveOptions blocked.hpp:630-636)
 * ------------------------------------------------------------------------- */
enum {
    CF_MODE_ATOMIC = 0,        /* in-tile fixed order, tile-shared nodes via fp64 RED */
    CF_MODE_DETERMINISTIC = 1  /* tile partials merged per node in ascending tile order
                                  (merge_blocks blocked.hpp:502-515): bit-reproducible */
};
enum {
    CF_NODE_ORDER_GIVEN = 0,   /* keep the caller's node numbering */
    CF_NODE_ORDER_RCM = 1,     /* rcm_permutation (reorder.hpp:127-148) */
    CF_NODE_ORDER_TILE = 2     /* first touch in tile order (device locality) */
};
enum {
    CF_ELEM_ORDER_GIVEN = 0,   /* tiles are contiguous chunks of the given element order */
    CF_ELEM_ORDER_MORTON = 1,  /* chunks of the Morton order of element centroids */
    CF_ELEM_ORDER_MIN_NODE = 2 /* chunks of the order by smallest (RCM) node label */
};
enum {
    CF_GEOM_STORED = 0,        /* tiles carry the precomputed 11-double ElementGeom (default) */
    CF_GEOM_COORDS = 1         /* tiles carry slot coordinates; the kernel recomputes the element
                                  gradients/volume (tet_geometry geometry.hpp:50-79, bitwise: same
                                  IEEE operations): ~40 % of the HBM bytes and device memory */
};
enum {
    CF_PARTITION_RCB = 0,      /* recursive coordinate bisection along the longest axis */
    CF_PARTITION_GIVEN = 1,    /* part_of_element supplied (load_partmap partition.hpp:424-445) */
    CF_PARTITION_GRAPH = 2     /* the reference's greedy graph partitioner over the virtual-element
                                  augmented dual graph (cf_partition_graph; balance_tol 0.05) */
};

typedef struct cf_run_opts {
    int32_t device;            /* CUDA ordinal of this process's first rank */
    int32_t mode;              /* CF_MODE_* */
    int32_t node_order;        /* CF_NODE_ORDER_* */
    int32_t elem_order;        /* CF_ELEM_ORDER_* */
    int32_t tile_elems;        /* elements per tile (0 = default 384) */
    const int32_t* tile_of_element; /* optional explicit block map (BlockPlan semantics,
                                       blocked.hpp:79-93); overrides elem_order/tile_elems */
    int32_t n_tiles_given;     /* tiles in tile_of_element */
    int32_t fast_math;         /* reserved, must be 0: kernels are built without FMA contraction
                                  (-fmad=false) so results are bitwise the reference's. An
                                  FMA-contracted build of the whole library is an opt-in
                                  (csrc/Makefile FMA=1: +2.6 % at cfg5, 2.8e-16 from the oracle) */
    /* domain decomposition (paper 4.1.1; two_level_decompose partition.hpp:377-422) */
    int32_t world_size;        /* ranks in the job (1 = single GPU) */
    int32_t rank;              /* this process's first rank */
    int32_t local_ranks;       /* ranks hosted by this process (1, or world_size for the
                                  in-process transport, see cf_comm_*) */
    int32_t partition;         /* CF_PARTITION_* */
    const int32_t* part_of_element; /* [n_elems] when CF_PARTITION_GIVEN */
    void* comm;                /* cf_comm* for world_size > local_ranks, else NULL */
    int32_t geometry;          /* CF_GEOM_* (0 = stored element geometry) */
} cf_run_opts;

typedef struct cf_plan cf_plan;
typedef struct cf_comm cf_comm;

/* Stats after stepping (SolverState fem.hpp:14-20, SolveResult blocked.hpp:638-647) */
typedef struct cf_stats {
    double time;
    double dt;                 /* last step's dt */
    int64_t step_index;
    int64_t clamp_steps;
    double loop_seconds;       /* device time of the stepping calls (CUDA events) */
    double static_dt;          /* local_static_dt (blocked.hpp:340-350), 0 if dynamic */
    int32_t dynamic_dt;
    int32_t n_tiles;           /* tiles (cache blocks) of this process's ranks */
    int64_t n_elems_local;     /* elements stepped by this process */
    int64_t n_nodes_local;
    int64_t total_slots;       /* Σ tile node counts (BlockPlan::total_local_nodes :85) */
    int64_t n_shared_nodes;
    int64_t n_ghost_nodes;
    int64_t device_bytes;      /* resident plan + state bytes */
    int64_t bytes_per_step;    /* canonical algorithmic bytes */
    int64_t launches_per_step; /* kernels launched per step */
    int64_t tile_bytes_per_launch; /* this layout's tile-kernel bytes per launch: blobs + slot T
                                      reads + 16 B of output per slot (partial or T + slot copy) */
    int64_t update_bytes_per_step; /* merge + update kernel's algorithmic bytes per step: per merged
                                      node its record (32 B), T read + write (16 B), and per partial
                                      the 16 B read + the 8 B slot-copy write */
    int64_t n_nodes_global;    /* nodes / elements of the whole mesh */
    int64_t n_elems_global;
    int32_t device_setup;      /* 1: the plan was built by the device setup pipeline */
} cf_stats;

/* ---------------------------------------------------------------------------
 * Entry points
 * ------------------------------------------------------------------------- */
int cf_abi_version(void);
int cf_last_error(char* buf, size_t len);

/* build_worker_model (blocked.hpp:156-361) + finalize_mesh (mesh.hpp:148-207) +
 * pair_sister_facets (mesh.hpp:456-478) + init_worker_fields (blocked.hpp:419-436):
 * validates the mesh and setup, builds tiles, uploads, sets T0 like
 * initial_temperatures (blocked.hpp:396-417) and refreshes the ambient. */
int cf_plan_create(const cf_mesh_desc* mesh, const cf_setup_desc* setup,
                   const cf_run_opts* opts, cf_plan** out);
int cf_plan_destroy(cf_plan* plan);

/* init_worker_fields (blocked.hpp:419-436) from a host global field [n_nodes]
 * + the pre-loop refresh_ambient (blocked.hpp:669); resets time/step/clamps. */
int cf_set_temperature(cf_plan* plan, const double* T_host);

/* n_steps × blocked_step (blocked.hpp:542-550). t_end > 0 caps each dt at
 * t_end - time and turns steps past t_end into no-ops (solve_serial :674-677);
 * t_end <= 0 is the max_steps mode (t_remaining = 0). No host sync inside. */
int cf_step(cf_plan* plan, int64_t n_steps, double t_end);

/* solve_serial's loop (blocked.hpp:671-684) with the output_every series:
 * runs until max_steps (>0) or setup.t_end; series written as (t, Tmin, Tmax)
 * triples into series[3*series_cap]; *n_series receives the count. */
int cf_solve(cf_plan* plan, int64_t max_steps, double* series, int64_t series_cap,
             int64_t* n_series);

/* Gather into global T, H (blocked.hpp:686-691); H = enthalpy(T) per region.
 * Either pointer may be NULL. Only nodes of this process's ranks are written. */
int cf_get_fields(cf_plan* plan, double* T_host, double* H_host);
int cf_get_stats(cf_plan* plan, cf_stats* out);

/* Device-resident access for benchmarks: current T buffer of local rank `r`
 * (rank-local node order) and its size. */
int cf_device_temperature(cf_plan* plan, int32_t local_rank, double** dptr, int64_t* n);

/* SolverConfig::dt_safety (material.hpp:157): rescales the static dt
 * (blocked.hpp:347) or the dynamic bound factor without rebuilding the plan. */
int cf_set_dt_safety(cf_plan* plan, double dt_safety);

/* Makes the next cf_step calls replay a CUDA graph of `steps_per_graph` steps. */
int cf_enable_graph(cf_plan* plan, int64_t steps_per_graph);

/* Runs n_steps real steps with CUDA events between the phases of each step
 * on the plan's stream; ms_out[4] = mean ms per step of {tile (assemble),
 * pack, exchange, update (merge+update)} summed over local ranks. */
int cf_time_phases(cf_plan* plan, int64_t n_steps, double* ms_out);

/* Largest eigenvalue of M_L^-1 (K + H_bc + H_if) at uniform reference
 * properties by power iteration on the device (setup utility: BASELINE's
 * "0.9x the explicit stability limit" is 0.9*2/lambda_max). Also returns the
 * reference Eq. 13 bound min_e rho c l^2/k (fem.hpp:83-85). */
int cf_estimate_lambda_max(cf_plan* plan, int32_t iterations, uint64_t seed,
                           double* lambda_max, double* eq13_min);

/* Tile-size autotuner: the recast of autotune_block_count / choose_block_count /
 * default_block_candidates (blocked.hpp:558-623). The reference tunes the CPU
 * cache-block count; on the B200 the knob is elements per tile (one tile per
 * CTA). Each candidate builds a plan (opts with tile_elems = candidate), steps
 * trial_steps from the setup's initial field twice and keeps the better device
 * time; a candidate whose tiles do not fit shared memory times +inf. */
typedef struct cf_tune_report {
    int32_t n_candidates;
    int32_t chosen;             /* tile_elems with the smallest time (first wins ties) */
    double overhead_fraction;   /* tune wall time / (tune wall + projected run), 0 if not projected */
} cf_tune_report;
int cf_autotune_tiles(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts,
                      const int32_t* candidates, int32_t n_candidates, int32_t trial_steps,
                      double projected_total_steps, double* seconds_out, cf_tune_report* out);
/* argmin of seconds, the first (smallest-index) candidate wins ties */
int cf_choose_tile_elems(const int32_t* candidates, const double* seconds, int32_t n, int32_t* chosen);
/* default candidates: multiples of 32 of the form 6*2^k (Morton chunks that are cell
 * boxes on structured meshes) from 192 to 1536, keeping at least 148 tiles; returns the count */
int cf_default_tile_candidates(int64_t n_elems, int32_t* out, int32_t cap, int32_t* count);

/* Multi-rank transport. NCCL across processes (one rank per GPU): rank 0
 * calls cf_comm_unique_id, shares the 128 bytes, every rank calls
 * cf_comm_create. world_size ranks in one process use the in-process
 * transport (local_ranks == world_size, comm == NULL). */
int cf_comm_unique_id(uint8_t out[128]);
int cf_comm_create(int32_t world_size, int32_t rank, int32_t device,
                   const uint8_t unique_id[128], cf_comm** out);
int cf_comm_destroy(cf_comm* comm);

/* Host-staged transport: the exchange_and_merge payload moves
 * through caller-supplied callbacks instead of NCCL, e.g. over a gloo / MPI / TCP
 * process group. Use it where NCCL cannot run: several rank processes sharing one
 * GPU (NCCL refuses duplicate devices) or hosts without a GPU interconnect. Each
 * step the pack kernel's send buffer is copied to pinned host memory, `sendrecv`
 * moves every neighbour's payload (one paired round, the edge-colouring stages of
 * S:441-449 collapsed), and the received payload is copied back before the update.
 * `allreduce` combines per-rank scalars (dynamic-dt bound: min; clamp flag and the
 * series' T_max: max; T_min: min) in place over all ranks. A nonzero callback
 * return fails the step with CF_PROTOCOL. Steps are host-synchronous (no CUDA
 * graphs). The callbacks are called from the thread that calls cf_step. */
typedef struct cf_host_transport {
    void* ctx;
    int (*sendrecv)(void* ctx, int32_t n_peers, const int32_t* peers, const double* const* send,
                    const int64_t* send_len, double* const* recv, const int64_t* recv_len);
    int (*allreduce)(void* ctx, double* values, int64_t count, int32_t op); /* op: CF_REDUCE_* */
} cf_host_transport;
enum { CF_REDUCE_MIN = 0, CF_REDUCE_MAX = 1 };
int cf_comm_create_host(int32_t world_size, int32_t rank, int32_t device,
                        const cf_host_transport* transport, cf_comm** out);

/* Peer-memory transport (NVLink 5 / NVSwitch P2P, one rank process per GPU): no library
 * collective on the data path. Every rank exports one device window (CUDA IPC) holding a
 * control block and its receive buffer for two step parities; `bootstrap` is used once per
 * plan to exchange the window handles (and once at cf_plan_destroy as a barrier, so a window
 * is unmapped everywhere before its owner frees it). Each step (SPEC S:450-458
 * exchange_and_merge): the pack kernel stores every neighbour's [c(shared) | r(shared) |
 * T(external)] payload straight into that neighbour's window and its last CTA raises this
 * rank's step flag there (system-scope release); the receiver's stream waits on its
 * neighbours' flags (cuStreamWaitValue32 -- no kernel spins on another rank) before the
 * update. Two parities suffice: a rank writes exchange k+2 only after its update k+1, which
 * waited for the neighbour's flag k+1, raised after the neighbour's update k read parity k.
 * The scalar reductions (dynamic-dt bound, clamp flag, series T_min / T_max) are all-to-all
 * stores into the control blocks. Steps stay asynchronous; CUDA graphs are not used (the
 * waited flag value changes every step). Limits: world_size <= 64, <= 32 neighbours per rank,
 * local_ranks == 1. Rank processes sharing one GPU work too (the windows are then local
 * memory), which is how the 1-GPU test pool exercises it. Destroy the plan before the comm. */
int cf_comm_create_peer(int32_t world_size, int32_t rank, int32_t device,
                        const cf_host_transport* bootstrap, cf_comm** out);

/* ---------------------------------------------------------------------------
 * Host utilities (no GPU needed) — the setup pipeline on either side of the path
 * ------------------------------------------------------------------------- */

/* rcm_permutation (reorder.hpp:127-148) over build_node_graph (:17-24):
 * new_of_old[n_nodes]. seed < 0 = pseudo-peripheral start per component. */
int cf_rcm_permutation(const cf_mesh_desc* mesh, int32_t seed, int32_t* new_of_old);
/* The same permutation computed on the B200 `device` (the RCM pass of the plan builder):
 * node graph built on the device from the tets, level-synchronous Cuthill-McKee in which each
 * level's order is (first-discovering parent position, degree, id) -- equal to rcm_permutation
 * element for element. Used by cf_plan_create for CF_NODE_ORDER_RCM. */
int cf_rcm_permutation_device(const cf_mesh_desc* mesh, int32_t seed, int32_t device, int32_t* new_of_old);
/* bandwidth (reorder.hpp:41-48); new_of_old NULL = identity. */
int cf_bandwidth(const cf_mesh_desc* mesh, const int32_t* new_of_old, int64_t* out);

/* finalize_mesh (mesh.hpp:148-207): orientation fix written to tets_out
 * [4E] (may alias nothing), facet owners to owner_out [F]. */
int cf_finalize_mesh(const cf_mesh_desc* mesh, int32_t* tets_out, int32_t* owner_out);

/* pair_sister_facets (mesh.hpp:456-478): returns the pair count; fills up to
 * cap triples (facet, sister element, contact) when out != NULL. */
int cf_pair_sister_facets(const cf_mesh_desc* mesh, int32_t* out, int64_t cap, int64_t* n_pairs);

/* Recursive coordinate bisection along the longest axis: part_of_element[E]. */
int cf_partition_rcb(const cf_mesh_desc* mesh, int32_t parts, int32_t* part_of_element);

/* Graph partitioning for unstructured decoupled meshes (paper 4.1.1): the reference's greedy
 * graph-growing partitioner (partition_graph partition.hpp:134-232) over the element dual graph
 * (build_dual_graph mesh.hpp:119-126), with augment != 0 first gluing the decoupled regions by one
 * zero-weight virtual element per cast-side interface pair (augment_virtual_elements
 * partition.hpp:43-91; partition_elements :236-241). Equal to the reference's partition. */
int cf_partition_graph(const cf_mesh_desc* mesh, int32_t parts, double balance_tol, int32_t augment,
                       int32_t* part_of_element);
/* partition_metrics (partition.hpp:250-272): edge cut and imbalance over the dual graph,
 * neighbor_counts[parts]; count_split_interface_pairs (:276-283). Any output may be NULL. */
int cf_partition_metrics(const cf_mesh_desc* mesh, const int32_t* part_of_element, int32_t parts,
                         int64_t* edge_cut, double* imbalance, int32_t* neighbor_counts,
                         int64_t* split_interface_pairs);

/* The tiles a plan would build (element -> tile map, in the plan's tile
 * order; for rank `rank` of a world of `world_size`, -1 for other ranks'
 * elements). Lets the CPU oracle replay the exact BlockPlan. */
int cf_tile_map(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts,
                int32_t* tile_of_element, int32_t* n_tiles);

/* The exchange plan of rank `rank` (classify_nodes partition.hpp:305-367 +
 * SPEC exchange_and_merge S:450-458), as global node ids. Per neighbour k
 * (ascending rank nbr_rank[k]): shared nodes (ascending global id; the c and r
 * partials travel in this order) and external nodes whose pre-update T flows
 * to / from it. Two-phase: NULL arrays return the sizes in counts[3*k..3*k+2]
 * (shared, ext_to, ext_from) after *n_nbrs; then pass arrays of those totals. */
int cf_exchange_plan(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts,
                     int32_t* n_nbrs, int32_t* nbr_rank, int64_t* counts, int32_t* shared, int32_t* ext_to,
                     int32_t* ext_from);

/* Synthetic fixtures (bench module S:502-519), structured Kuhn 6-tet cubes.
 * kind: 0 = single-region cube, all faces tag "outer";
 *       1 = casting: sphere of radius `radius` (cell-centre test) in a mould
 *           box, interface nodes duplicated, tags outer / cast_if / mold_if,
 *           contact (cast_if, mold_if).
 * jitter: interior grid points moved by U(±jitter·h) per coordinate (seeded
 * per grid point). perm_seed != 0 permutes element and node numbering.
 * Two-phase call: pass NULL arrays to get sizes, then allocated arrays. */
typedef struct cf_fixture {
    int32_t n_nodes, n_elems, n_facets;
    double* coords;      /* [3N] */
    int32_t* tets;       /* [4E] */
    int32_t* region;     /* [E] */
    int32_t* facets;     /* [3F] */
    int32_t* facet_tag;  /* [F] tag ids: 0 outer, 1 cast_if, 2 mold_if */
    int32_t* node_grid;  /* [N] optional: linear grid-point index of each node */
} cf_fixture;
int cf_generate_fixture(int32_t kind, int32_t n, double radius, double jitter, uint64_t seed,
                        uint64_t perm_seed, cf_fixture* out);

/* A plan over a fixture generated on the device (the same mesh cf_generate_fixture
 * returns, perm_seed 0): the mesh never exists in host memory (cfg5: 805 M tets). The
 * setup's tags are the fixture's ("outer", "cast_if", "mold_if"); T0 is the material
 * initial temperature of each node's region plus U(-t0_noise, t0_noise) keyed by grid point
 * with noise_seed (cf_counter_uniform), unless setup->initial_T is given. */
typedef struct cf_fixture_spec {
    int32_t kind, n;        /* 0 cube, 1 casting; n^3 cells */
    double radius, jitter;
    uint64_t seed, perm_seed;  /* perm_seed must be 0 */
    double t0_noise;
    uint64_t noise_seed;
    int32_t rcm;            /* 1: node numbering permuted by the RCM pass (permute_mesh(m,
                               rcm_permutation(m)), reorder.hpp:127-163), like an RCM-reordered
                               input mesh */
} cf_fixture_spec;
int cf_plan_create_fixture(const cf_fixture_spec* fx, const cf_setup_desc* setup,
                           const cf_run_opts* opts, cf_plan** out);

/* Counter-based uniform noise U(lo, hi) keyed by (seed, key) — T0 noise
 * keyed by grid point so it is independent of numbering. */
int cf_counter_uniform(uint64_t seed, const int64_t* keys, int64_t n, double lo, double hi,
                       double* out);

/* Test instrumentation: FNV-1a digests of one rank's tiled plan, one per plan array
 * (scalars, tile_meta, tile_border, tile_slot_off, blob_off, elem_off, staged blob sections,
 * tets_ord, elem_global, slot_node, local_global, node_region, node_dir, merge_off, merge_idx,
 * shared_list, neighbour lists, exchange tables), CF_DIGEST_LEN entries. Host plan builder. */
#define CF_DIGEST_LEN 24
int cf_plan_digest(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts,
                   int32_t rank, uint64_t* digest);
/* The same digests from the device setup pipeline (tets_ord is not kept there: its entry is
 * the digest of an empty array), and the device RCB partition. Need a B200. */
int cf_plan_digest_device(const cf_mesh_desc* mesh, const cf_setup_desc* setup, const cf_run_opts* opts,
                          int32_t rank, uint64_t* digest);
int cf_partition_rcb_device(const cf_mesh_desc* mesh, int32_t parts, int32_t* out);

/* ---------------------------------------------------------------- text formats
 * The reference's file formats either side of the step (same tokenizer, number
 * syntax, sections, defaults and error messages; CF_PARSE messages carry
 * "line N: "). Parsed objects own their arrays; *_view fills a descriptor that
 * points into them (valid until *_free). *_format writes NUL-terminated text
 * into buf (truncated to cap-1) and returns the full length in *len. */
typedef struct cf_text_mesh cf_text_mesh;
typedef struct cf_text_setup cf_text_setup;

/* parse_mesh mesh.hpp:256-325 ("femesh 1"; nodes / tets / facets / contact
 * sections), including finalize_mesh: a rejected mesh is CF_VALIDATION
 * "mesh validation failed: ..."; the view's tets are oriented like the
 * reference's finalized Mesh. */
int cf_mesh_parse(const char* text, int64_t len, cf_text_mesh** out);
int cf_mesh_view(const cf_text_mesh* m, cf_mesh_desc* out);
void cf_mesh_free(cf_text_mesh* m);
/* write_mesh mesh.hpp:327-343 (coordinates %.17g) */
int cf_mesh_format(const cf_mesh_desc* mesh, char* buf, int64_t cap, int64_t* len);
/* binary fast path (this repo's format "CFMESHB1": counts, then the raw arrays and tag
 * strings; little-endian) for meshes too large for text; parse validates and orients like
 * cf_mesh_parse. format: *len = bytes needed; buf (if non-NULL) must hold them. */
int cf_mesh_parse_binary(const void* data, int64_t len, cf_text_mesh** out);
int cf_mesh_format_binary(const cf_mesh_desc* mesh, void* buf, int64_t cap, int64_t* len);

/* parse_config material.hpp:186-345: [material r] rho c k latent_heat solidus
 * liquidus T0 / [bc tag] kind T q h T_inf / [interface a b] h h_time h_temp /
 * [solver] safety t_end output_every; tables are x:y pairs or one constant.
 * The view's initial_T is NULL (per-region T0). */
int cf_config_parse(const char* text, int64_t len, cf_text_setup** out);
int cf_config_view(const cf_text_setup* s, cf_setup_desc* out);
void cf_config_free(cf_text_setup* s);

/* load_partmap / write_partmap partition.hpp:424-449: one part id per element */
int cf_partmap_parse(const char* text, int64_t len, int32_t n_elems, int32_t* parts_out, int32_t* part_count);
int cf_partmap_format(const int32_t* parts, int32_t n, char* buf, int64_t cap, int64_t* len);

#ifdef __cplusplus
}
#endif
#endif /* CASTFEM_B200_H */
