// cf_internal.hpp — host-side types of the B200 castfem step (not part of the ABI).
//
// The host layer keeps the reference's setup semantics (mesh validation,
// sister pairing, facet resolution, Dirichlet lists, static dt — all cited in
// the .cpp files) and lays the result out for the device: element tiles are
// the paper's cache blocks (BlockPlan, blocked.hpp:79-93) recast as
// thread-block tiles.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <memory>
#include <utility>
#include <vector>

#include "../../include/castfem_b200.h"
#include "cf_tileblob.hpp"

namespace cfb {

// allocator that leaves trivially constructible elements uninitialised, so big
// host staging buffers are first touched by the parallel loops that fill them
template <class T>
struct UninitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = UninitAlloc<U>;
    };
    UninitAlloc() = default;
    template <class U>
    UninitAlloc(const UninitAlloc<U>&) {}
    template <class U>
    void construct(U* p) { ::new ((void*)p) U; }
    template <class U, class... A>
    void construct(U* p, A&&... a) { ::new ((void*)p) U(std::forward<A>(a)...); }
};

// Exception carrying a CF_* status; mapped at the C-ABI edge.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

// CF_TRACE_SETUP=1: host setup stage times on stderr (diagnostics only).
void trace_stage(const char* name);

void set_last_error(const std::string& msg);

// Per-element geometry (TetGeometry geometry.hpp:36-41).
struct Geom {
    double vol;
    double g[4][3];
    double min_edge, max_edge;
};
// tet_geometry geometry.hpp:48-77 (same operation order; -ffp-contract=off).
bool tet_geometry(const double* p0, const double* p1, const double* p2, const double* p3, Geom& g);
double triangle_area(const double* a, const double* b, const double* c);
void triangle_centroid(const double* a, const double* b, const double* c, double* out);

// Mesh after finalize_mesh (mesh.hpp:148-207).
struct MeshData {
    int32_t N = 0, E = 0, F = 0;
    const double* coords = nullptr;   // caller's [3N]
    std::vector<int32_t, UninitAlloc<int32_t>> tets;        // oriented [4E]
    const int32_t* region = nullptr;  // caller's [E]
    const int32_t* facets = nullptr;  // caller's [3F]
    const int32_t* facet_tag = nullptr;
    std::vector<int32_t> owner;       // [F]
    std::vector<int32_t> node_region; // [N]
    std::vector<std::string> tags;
    std::vector<int32_t> contacts;    // [2C]
    int32_t region_count = 0;
    std::vector<double> region_min_edge;  // per region: min element min_edge (static dt, Eq. 13)
    const double* pos(int32_t n) const { return coords + 3 * (size_t)n; }
    Geom geometry(int64_t e) const;       // tet_geometry of the oriented element
};

// finalize_mesh: orientation, degeneracy, regions, facet owners, per-region
// minimum edge. Geometry is recomputed per element where needed (build_rank_plan
// only for the rank's own elements), so no O(E) geometry array is held.
void finalize_mesh(const cf_mesh_desc* d, MeshData& m);

struct Pair {
    int32_t facet, sister, contact;
};
// pair_sister_facets mesh.hpp:456-478.
std::vector<Pair> pair_sister_facets(const MeshData& m);

// Node adjacency CSR (build_node_graph reorder.hpp:17-24; sorted, deduplicated).
struct Graph {
    int32_t n = 0;
    std::vector<int64_t> off;
    std::vector<int32_t> adj;
    int32_t degree(int32_t v) const { return (int32_t)(off[v + 1] - off[v]); }
};
Graph build_node_graph(int32_t N, int32_t E, const int32_t* tets);
// rcm_permutation reorder.hpp:127-148 (exact order reproduction).
std::vector<int32_t> rcm_permutation(const Graph& g, int32_t seed);
int64_t bandwidth(const Graph& g, const int32_t* new_of_old);
// The same permutation computed on the B200 (cf_rcm.cu): device node graph + level-synchronous
// Cuthill-McKee with first-discoverer claims; equal to rcm_permutation.
std::vector<int32_t> rcm_permutation_device(int32_t N, int64_t E, const int32_t* tets, int32_t seed, int device);
bool cuda_device_present();

// Recursive coordinate bisection along the longest axis.
std::vector<int32_t> partition_rcb(const MeshData& m, int32_t parts);

// Graph partitioning of decoupled meshes (cf_partition.cpp): partition_graph partition.hpp:134-232
// over the dual graph (build_dual_graph mesh.hpp:119-126), optionally augmented with virtual
// elements (augment_virtual_elements partition.hpp:43-91); quality metrics :243-283.
struct PartitionQuality {
    int64_t edge_cut = 0;
    double imbalance = 1.0;
    std::vector<int32_t> neighbor_counts;
};
Graph dual_graph(const MeshData& m);
std::vector<int32_t> partition_graph(const Graph& g, const std::vector<int32_t>& weights, int32_t k, double tol);
std::vector<int32_t> partition_elements(const MeshData& m, int32_t k, double tol, bool augment);
PartitionQuality partition_metrics(const MeshData& m, const int32_t* part, int32_t k);
int64_t count_split_interface_pairs(const MeshData& m, const int32_t* part);

// Fixtures (SPEC bench module S:502-519).
struct FixtureSizes {
    int32_t N, E, F;
};
void generate_fixture(int kind, int n, double radius, double jitter, uint64_t seed, uint64_t perm_seed,
                      cf_fixture* out);
double counter_uniform(uint64_t seed, uint64_t key);

// ---------------------------------------------------------------- setup
// Device-facing material record (MaterialTable material.hpp:53-124).
constexpr int kMaxRegions = 16;
constexpr int kMaxTablePts = 1024;
constexpr int kMaxFacetKinds = 64;

struct DevTable {    // into the params table pool; n == 1 constant
    int32_t n, off;
};
struct DevMaterial {
    double rho, latent, solidus, liquidus, ref;
    double c0, k0;          // constant values (n == 1)
    double range_lo, range_hi;
    double T0;              // initial_temperature (lambda_max estimate only)
    DevTable c, k;
    int32_t cum_off;        // cumulative enthalpy at breakpoints (non-constant c)
    int32_t has_phase;
};
// A facet "kind": flux BC parameters or an interface coefficient.
struct DevFacetKind {
    int32_t interface;      // 0 flux, 1 interface
    int32_t var;            // CF_VAR_*
    double q, h, t_inf;
    DevTable htab;
};
struct DevParams {
    int32_t n_materials;
    int32_t temp_dep;       // any non-constant c/k table -> dynamic dt
    int32_t finite_range;
    int32_t n_kinds;
    double dt_safety;
    double static_dt;
    DevMaterial mat[kMaxRegions];
    DevFacetKind kind[kMaxFacetKinds];
    DevTable dir_tab[kMaxFacetKinds];   // Dirichlet fixed_T(t) tables by dirichlet id
    double pool[kMaxTablePts];          // table x/y values and cumulative enthalpy
};

// Resolved setup shared by every rank.
struct SetupData {
    DevParams P{};
    std::vector<int32_t> facet_kind;    // [F]: kind id, -1 - dirichlet id for fixed BCs
    std::vector<int32_t> dir_of_node;   // [N]: dirichlet id (lowest tag) or -1
    std::vector<double> T0;             // [N] initial temperatures (initial_temperatures :396-417)
    std::vector<Pair> pairs;
    std::vector<int32_t> pair_of_facet; // [F]
    bool temp_dep = false;
    double min_bound = 0;               // min_e rho c l^2 / k before the safety factor
    bool static_dt_only = false;        // node arrays not built here (device setup)
    std::vector<int32_t> kind_of_tag;   // [tags] facet kind per tag (-1 - dirichlet id), INT32_MIN unused
};
void resolve_setup(const MeshData& m, const cf_setup_desc* s, SetupData& out);
// the same with the element-region facts given (device meshes: m holds only the facet part)
// and, node_arrays false, without the O(N) dir_of_node / T0 arrays
struct RegionUse {
    int32_t first_bad_region = -1;  // region of the first element whose region has no material
    uint32_t mask = 0;              // regions in use
};
void resolve_setup_impl(const MeshData& m, const cf_setup_desc* s, SetupData& out, const RegionUse* ru,
                        bool node_arrays);
double pl_eval(const DevParams& P, const DevTable& t, double x);
double enthalpy(const DevParams& P, const DevMaterial& m, double T);

// ---------------------------------------------------------------- tiles
constexpr int kMaxTileElems = 2048;

// One rank's tiled plan (host copy, uploaded as-is). Element data lives in
// per-tile blobs (cf_tileblob.hpp) fetched by one TMA bulk copy per tile.
struct RankPlan {
    int32_t rank = 0;
    int32_t n_local = 0, n_ghost = 0;      // local nodes, then ghost (external) nodes
    std::vector<int32_t> local_global;     // [n_local + n_ghost] global ids
    std::vector<uint8_t> node_region;      // [n_local]
    std::vector<int8_t> node_dir;          // [n_local] dirichlet id or -1 (empty if none)
    // tiles
    int32_t n_tiles = 0;
    std::vector<TileMeta> tile_meta;       // [n_tiles] ne, ns, nf, ncsr
    std::vector<uint8_t> tile_border;      // [n_tiles] holds a rank-shared node (multi-rank)
    std::vector<int32_t> tile_slot_off;    // [n_tiles+1]
    std::vector<int64_t> blob_off;         // [n_tiles+1] byte offsets into blob
    std::vector<uint8_t, UninitAlloc<uint8_t>> blob;  // host staging: tiles' [conn, bytes) sections at rest_off
    std::vector<int64_t> rest_off;         // [n_tiles+1] offsets into blob (after a leading pad)
    int64_t blob_bytes = 0;                // device blob size (blob_off[n_tiles])
    std::vector<int64_t> elem_off;         // [n_tiles+1] first element of each tile (tile order)
    std::vector<int32_t, UninitAlloc<int32_t>> tets_ord;    // [4 E_r] oriented tets, local ids, tile order
    std::vector<double, UninitAlloc<double>> coords_local;  // [3 n_local] node coordinates
    bool coords = false;                   // CF_GEOM_COORDS layout (cf_tileblob.hpp)
    int32_t max_slots = 0, max_elems = 0, max_facets = 0;
    int64_t max_blob = 0;
    int64_t max_scratch = 0;               // coordinates layout: contribution scratch doubles
    std::vector<int32_t> elem_global;      // [E_r] tile order
    std::vector<int32_t> slot_node;        // [S] local node id
    int64_t n_bc_facets = 0, n_if_facets = 0;
    // merge: per local node, partial (slot) indices in ascending tile order
    std::vector<int32_t> merge_off;        // [n_local+1]
    std::vector<int32_t> merge_idx;        // [S]
    std::vector<int32_t> shared_list;      // local nodes needing a merge (touched by >1 tile or rank)
    int64_t n_private = 0;
    // multi-rank exchange
    struct Neighbor {
        int32_t rank;
        std::vector<int32_t> shared;       // local ids, ascending global id
        std::vector<int32_t> ext_to;       // local ids whose T the neighbor needs
        std::vector<int32_t> ext_from;     // ghost ids (local numbering) received from it
    };
    std::vector<Neighbor> nbrs;            // ascending rank
    std::vector<int32_t> node_shared;      // [n_local] shared index or -1
    std::vector<int32_t> shared_off;       // [n_shared+1]
    std::vector<int32_t> shared_src;       // -1 own, else c index into the recv buffer (ascending rank)
    std::vector<int32_t> shared_src_r;     // r index into the recv buffer
    std::vector<int64_t> send_off, recv_off; // per neighbor buffer offsets (doubles)
    std::vector<int32_t> ghost_src;        // [n_ghost] index into recv buffer
    int64_t send_len = 0, recv_len = 0;
    int64_t n_shared = 0;
};

struct TileCtx;
// environment knobs of the tile builder (CF_SLOT_ORDER, CF_SLOT_BANKS, CF_BANK_PASSES,
// CF_BANK_ITERS), read once per plan by both builders
void tile_env(TileCtx& c);

struct PlanOptions {
    int mode = CF_MODE_ATOMIC;
    int node_order = CF_NODE_ORDER_RCM;
    int elem_order = CF_ELEM_ORDER_MORTON;
    int tile_elems = 1024;
    int geometry = CF_GEOM_STORED;
    const int32_t* tile_of_element = nullptr;
    int32_t n_tiles_given = 0;
    int world_size = 1;
    const int32_t* part_of_element = nullptr;  // resolved (RCB or given)
};

// Builds rank `rank`'s tiles (build_worker_model blocked.hpp:156-361 recast).
void build_rank_plan(const MeshData& m, const SetupData& S, const PlanOptions& o,
                     const std::vector<int32_t>& node_label, int32_t rank, RankPlan& rp);

}  // namespace cfb
