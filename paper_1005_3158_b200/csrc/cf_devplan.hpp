// cf_devplan.hpp — the setup pipeline on the B200: mesh finalize, the
// fixture generator, setup resolution, RCM, recursive coordinate bisection and the tile
// builder run on the device, so a plan is built without the mesh ever existing in host
// memory (cfg5: 805 M tets, ~20 GB of mesh arrays). The per-tile logic is cf_tilepack.hpp,
// shared with the host builder (cf_plan.cpp), so both produce byte-identical plans
// (cf_plan_digest). Only O(facets) and O(tiles) metadata visit the host.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "cf_internal.hpp"

namespace cfb {

// the RCM pass over device-resident tets (cf_rcm.cu); new_of_old: device array [N]
void rcm_labels_device(int32_t N, int64_t E, const int32_t* tets, int32_t seed, cudaStream_t s, int32_t* new_of_old);

// device allocations owned by one object
struct DBuf {
    std::vector<void*> p;
    std::vector<size_t> sz;
    int64_t bytes = 0;
    template <class T>
    T* alloc(size_t n) {
        void* q = nullptr;
        const size_t b = (n ? n : 1) * sizeof(T);
        const cudaError_t e = cudaMalloc(&q, b);
        if (e != cudaSuccess)
            raise(CF_CUDA, std::string("device allocation of ") + std::to_string(b) + " B: " + cudaGetErrorString(e));
        p.push_back(q);
        sz.push_back(b);
        bytes += (int64_t)b;
        return (T*)q;
    }
    void free(const void* q) {
        for (size_t i = 0; i < p.size(); ++i)
            if (p[i] == q) {
                cudaFree(p[i]);
                bytes -= (int64_t)sz[i];
                p.erase(p.begin() + (long)i);
                sz.erase(sz.begin() + (long)i);
                return;
            }
    }
    void release() {
        for (void* q : p) cudaFree(q);
        p.clear();
        sz.clear();
        bytes = 0;
    }
    ~DBuf() { release(); }
};

// A finalized mesh resident on the device (Mesh mesh.hpp:45-80 after finalize_mesh :148-207).
struct DevMesh {
    int32_t N = 0, E = 0, F = 0;
    double* coords = nullptr;       // [3N]
    int32_t* tets = nullptr;        // [4E] oriented (n2/n3 swapped where the volume was negative)
    int32_t* region = nullptr;      // [E]
    int32_t* facets = nullptr;      // [3F]
    int32_t* node_region = nullptr; // [N]
    int32_t* node_grid = nullptr;   // [N] fixtures: grid point of each node (T0 noise key)
    std::vector<int32_t> h_facets, h_facet_tag, h_owner;  // O(F) host copies
    std::vector<std::string> tags;
    std::vector<int32_t> contacts;  // [2C]
    int32_t region_count = 0;
    uint32_t region_mask = 0;       // regions referenced (bit r, r < 32)
    int32_t max_region = -1;
    std::vector<double> region_min_edge;
    DBuf mem;
};

// upload + validate/orient on the device; any defect is re-diagnosed by the host finalize_mesh,
// which raises the reference's exact error
void devmesh_from_desc(const cf_mesh_desc* d, cudaStream_t s, DevMesh& m);
// generate_fixture on the device (perm_seed 0): same coordinates, numbering, tets, facets;
// rcm: then renumbered by the RCM pass (permute_mesh(m, rcm_permutation(m)), reorder.hpp:127-163)
void devmesh_fixture(int kind, int n, double radius, double jitter, uint64_t seed, bool rcm, cudaStream_t s,
                     DevMesh& m);

// resolved setup over a device mesh: tables, facet kinds, sister pairs on the host (O(F));
// Dirichlet node ids and T0 on the device (O(N))
struct DevSetup {
    SetupData S;                    // dir_of_node / T0 left empty
    int32_t* dir_of_node = nullptr; // [N] device, null if no Dirichlet facet
    double* T0 = nullptr;           // [N] device
    DBuf mem;
};
struct T0Noise {                    // T0 = material T0 + U(-amp, amp) keyed by node_grid (fixtures)
    double amp = 0;
    uint64_t seed = 0;
};
void resolve_setup_device(const DevMesh& m, const cf_setup_desc* s, const T0Noise& noise, cudaStream_t st,
                          DevSetup& out);

// partition_rcb on the device (same parts: (centroid coordinate, id) order per bisection)
void partition_rcb_device(const DevMesh& m, int32_t parts, cudaStream_t s, int32_t* part);

// One rank's plan built on the device: metadata on the host (RankPlan fields the launch
// configuration reads), the big arrays in device memory
struct DevRankPlan {
    RankPlan H;                     // n_tiles, tile_meta, tile_border, tile_slot_off, blob_off, n_local,
                                    // n_ghost, max_*, n_if/bc_facets, n_private, n_shared, nbrs,
                                    // send/recv offsets and lengths
    int64_t E_r = 0, S_tot = 0, n_shared_list = 0, merge_parts = 0;
    uint8_t* blob = nullptr;
    int32_t* slot_node = nullptr;
    int32_t* local_global = nullptr;
    uint8_t* node_region = nullptr;
    int8_t* node_dir = nullptr;
    int32_t* merge_off = nullptr;
    int32_t* merge_idx = nullptr;
    int32_t* shared_list = nullptr;
    int4* shared_rec = nullptr;
    int2* shared_rec2 = nullptr;
    int32_t* elem_global = nullptr; // [E_r] tile order (kept for cf_tile_map-style queries)
    // multi-rank exchange tables (device)
    int32_t *node_shared = nullptr, *shared_off = nullptr, *shared_src = nullptr, *shared_src_r = nullptr,
            *ghost_src = nullptr;
    DBuf mem;
};
void build_rank_plan_device(const DevMesh& m, const DevSetup& S, const PlanOptions& o, const int32_t* d_label,
                            const int32_t* d_part, int32_t rank, cudaStream_t s, DevRankPlan& out);

// the device plan's arrays downloaded into a host RankPlan (test instrumentation: plan digests)
void download_dev_rank_plan(const DevRankPlan& p, bool tdep, bool coords, cudaStream_t s, RankPlan& rp);

}  // namespace cfb
