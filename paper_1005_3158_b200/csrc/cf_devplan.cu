// cf_devplan.cu — the setup pipeline on the B200 (see cf_devplan.hpp).
//
// Reference semantics (paths relative to /root/reference/proj/include/castfem/):
//   finalize_mesh            mesh.hpp:148-207 (orientation, degeneracy, node regions, owners)
//   generate_fixture         this repo's Kuhn-split casting generator (cf_mesh.cpp), same ids
//   resolve_facet_tag etc.   blocked.hpp:127-149, 250-263, 340-350 (resolve_setup, cf_plan.cpp)
//   partition (RCB)          SURVEY 8(e): recursive coordinate bisection along the longest axis
//   build_worker_model       blocked.hpp:156-361 recast as tiles (build_rank_plan, cf_plan.cpp)
// Every stage reproduces the host implementation exactly; the per-tile work is the shared
// cf_tilepack.hpp code, one tile per thread.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <cstring>
#include <numeric>

#include "cf_devplan.hpp"
#include "cf_physics.cuh"
#include "cf_tilepack.hpp"

namespace cfb {
namespace {

#define DP_CHECK(x)                                                                                      \
    do {                                                                                                 \
        cudaError_t e_ = (x);                                                                            \
        if (e_ != cudaSuccess) raise(CF_CUDA, std::string("device setup: ") + #x + ": " + cudaGetErrorString(e_)); \
    } while (0)

inline int grid_of(int64_t n, int block = 256) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(148 * 32, (n + block - 1) / block));
}
#define GRID_STRIDE(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

template <class T>
void h2d(T* d, const T* h, size_t n, cudaStream_t s) {
    if (n) DP_CHECK(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
void d2h(T* h, const T* d, size_t n, cudaStream_t s) {
    if (n) DP_CHECK(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    DP_CHECK(cudaStreamSynchronize(s));
}
template <class T>
T read1(const T* d, cudaStream_t s) {
    T v;
    d2h(&v, d, 1, s);
    return v;
}

// ---- CUB wrappers (temporary storage per call)
template <class K, class V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int bits, cudaStream_t s) {
    if (n <= 0) return;
    size_t tb = 0;
    DP_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, bits, s));
    DBuf T;
    void* tmp = T.alloc<uint8_t>(tb);
    DP_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, kin, kout, vin, vout, n, 0, bits, s));
    DP_CHECK(cudaStreamSynchronize(s));
}
template <class K>
void sort_keys(const K* kin, K* kout, int64_t n, int bits, cudaStream_t s) {
    if (n <= 0) return;
    size_t tb = 0;
    DP_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tb, kin, kout, n, 0, bits, s));
    DBuf T;
    void* tmp = T.alloc<uint8_t>(tb);
    DP_CHECK(cub::DeviceRadixSort::SortKeys(tmp, tb, kin, kout, n, 0, bits, s));
    DP_CHECK(cudaStreamSynchronize(s));
}
template <class In, class Out>
void excl_sum(const In* in, Out* out, int64_t n, cudaStream_t s) {  // out[n] = total (out sized n + 1)
    if (n <= 0) {
        DP_CHECK(cudaMemsetAsync(out, 0, sizeof(Out), s));
        return;
    }
    size_t tb = 0;
    DP_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out + 1, n, s));
    DBuf T;
    void* tmp = T.alloc<uint8_t>(tb);
    DP_CHECK(cudaMemsetAsync(out, 0, sizeof(Out), s));
    DP_CHECK(cub::DeviceScan::InclusiveSum(tmp, tb, in, out + 1, n, s));
    DP_CHECK(cudaStreamSynchronize(s));
}
// segmented ascending sort of int32 keys in place (segments [off[i], off[i+1]))
void seg_sort_keys(int32_t* keys, int64_t n, const int64_t* off, int64_t nseg, cudaStream_t s) {
    if (n <= 0 || nseg <= 0) return;
    DBuf T;
    int32_t* out = T.alloc<int32_t>(n);
    size_t tb = 0;
    DP_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, keys, out, n, nseg, off, off + 1, s));
    void* tmp = T.alloc<uint8_t>(tb);
    DP_CHECK(cub::DeviceSegmentedSort::SortKeys(tmp, tb, keys, out, n, nseg, off, off + 1, s));
    DP_CHECK(cudaMemcpyAsync(keys, out, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    DP_CHECK(cudaStreamSynchronize(s));
}

template <class T>
__global__ void k_fill(int64_t n, T* a, T v) {
    GRID_STRIDE(i, n) a[i] = v;
}

// order-preserving map of a double onto uint64 (and back)
__host__ __device__ __forceinline__ uint64_t dkey(double v) {
    uint64_t b;
    memcpy(&b, &v, 8);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double dval(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    memcpy(&v, &b, 8);
    return v;
}

// ------------------------------------------------------------------ finalize (mesh.hpp:148-207)
struct FinFlags {
    int32_t bad_coord;                  // non-finite coordinate
    unsigned long long bad_elem;        // first element failing index / repeat / region / degeneracy
    int32_t region_conflict, unreferenced, bad_facet_node, facet_error;
    int32_t max_region;
    uint32_t region_mask;
    unsigned long long region_min_edge[32];
};

__global__ void k_check_coords(int64_t n3, const double* c, FinFlags* f) {
    GRID_STRIDE(i, n3) if (!isfinite(c[i])) f->bad_coord = 1;
}

// index range, repeated node, negative region, orientation swap (tet_signed_volume < 0,
// mesh.hpp:170-172), degeneracy (tet_geometry geometry.hpp:66-69), per-region minimum edge
__global__ void k_orient(int64_t E, int32_t N, int32_t* tets, const int32_t* region, const double* X, FinFlags* f) {
    GRID_STRIDE(e, E) {
        int4 t = ((int4*)tets)[e];
        int32_t q[4] = {t.x, t.y, t.z, t.w};
        int code = 0;
        for (int a = 0; a < 4; ++a)
            if (q[a] < 0 || q[a] >= N) code = 1;
        if (!code)
            for (int a = 0; a < 4; ++a)
                for (int b = a + 1; b < 4; ++b)
                    if (q[a] == q[b]) code = 2;
        const int32_t rg = region[e];
        if (!code && rg < 0) code = 3;
        if (!code) {
            double p[4][3];
            for (int a = 0; a < 4; ++a)
                for (int k = 0; k < 3; ++k) p[a][k] = X[3 * (int64_t)q[a] + k];
            const double e1[3] = {p[1][0] - p[0][0], p[1][1] - p[0][1], p[1][2] - p[0][2]};
            const double e2[3] = {p[2][0] - p[0][0], p[2][1] - p[0][1], p[2][2] - p[0][2]};
            const double e3[3] = {p[3][0] - p[0][0], p[3][1] - p[0][1], p[3][2] - p[0][2]};
            const double c0 = e2[1] * e3[2] - e2[2] * e3[1];
            const double c1 = e2[2] * e3[0] - e2[0] * e3[2];
            const double c2 = e2[0] * e3[1] - e2[1] * e3[0];
            if ((e1[0] * c0 + e1[1] * c1 + e1[2] * c2) / 6.0 < 0) {
                const int32_t x = q[2];
                q[2] = q[3];
                q[3] = x;
                for (int k = 0; k < 3; ++k) {
                    const double y = p[2][k];
                    p[2][k] = p[3][k];
                    p[3][k] = y;
                }
                ((int4*)tets)[e] = make_int4(q[0], q[1], q[2], q[3]);
            }
            double g[4][3], vol, mn, mx;
            dev_tet_geometry(p, g, vol, mn, mx);
            const double eps = 1e-12 * mx * mx * mx;
            if (!(vol > eps)) code = 4;
            atomicMax(&f->max_region, rg);
            if (rg < 32) {
                atomicOr(&f->region_mask, 1u << rg);
                atomicMin(&f->region_min_edge[rg], (unsigned long long)__double_as_longlong(mn));
            }
        }
        if (code) atomicMin(&f->bad_elem, (unsigned long long)e);
    }
}

__global__ void k_node_region(int64_t E, const int32_t* tets, const int32_t* region, int32_t* nreg, FinFlags* f) {
    GRID_STRIDE(k, 4 * E) {
        const int32_t r = region[k >> 2];
        const int32_t old = atomicCAS(&nreg[tets[k]], -1, r);
        if (old != -1 && old != r) f->region_conflict = 1;
    }
}
__global__ void k_unreferenced(int64_t N, const int32_t* nreg, FinFlags* f) {
    GRID_STRIDE(n, N) if (nreg[n] < 0) f->unreferenced = 1;
}

// facet hash (sorted node triple); duplicate facets share the slot of the first (smallest id)
__device__ __forceinline__ void sort3d(int32_t* k) {
    int32_t t;
    if (k[0] > k[1]) { t = k[0]; k[0] = k[1]; k[1] = t; }
    if (k[1] > k[2]) { t = k[1]; k[1] = k[2]; k[2] = t; }
    if (k[0] > k[1]) { t = k[0]; k[0] = k[1]; k[1] = t; }
}
__device__ __forceinline__ uint64_t hash3d(const int32_t* k) {
    uint64_t h = (uint64_t)(uint32_t)k[0] * 0x9E3779B97F4A7C15ull;
    h ^= ((uint64_t)(uint32_t)k[1] + 0x7F4A7C159E3779B9ull) * 0xBF58476D1CE4E5B9ull;
    h ^= ((uint64_t)(uint32_t)k[2] + 0x94D049BB133111EBull) * 0xC2B2AE3D27D4EB4Full;
    h ^= h >> 29;
    return h;
}
__device__ __forceinline__ void fkey(const int32_t* facets, int32_t f, int32_t* k) {
    k[0] = facets[3 * (int64_t)f];
    k[1] = facets[3 * (int64_t)f + 1];
    k[2] = facets[3 * (int64_t)f + 2];
    sort3d(k);
}
__global__ void k_facet_nodes(int64_t F, int32_t N, const int32_t* facets, uint8_t* on, FinFlags* f) {
    GRID_STRIDE(i, 3 * F) {
        const int32_t n = facets[i];
        if (n < 0 || n >= N) f->bad_facet_node = 1;
        else on[n] = 1;
    }
}
__global__ void k_facet_insert(int64_t F, const int32_t* facets, int32_t* slot, uint64_t mask) {
    GRID_STRIDE(f, F) {
        int32_t k[3];
        fkey(facets, (int32_t)f, k);
        uint64_t h = hash3d(k) & mask;
        for (;;) {
            const int32_t cur = atomicCAS(&slot[h], -1, (int32_t)f);
            if (cur == -1) break;
            int32_t o[3];
            fkey(facets, cur, o);
            if (o[0] == k[0] && o[1] == k[1] && o[2] == k[2]) {
                atomicMin(&slot[h], (int32_t)f);
                break;
            }
            h = (h + 1) & mask;
        }
    }
}
__device__ __forceinline__ int32_t facet_find(const int32_t* facets, const int32_t* slot, uint64_t mask, const int32_t* k) {
    uint64_t h = hash3d(k) & mask;
    for (;;) {
        const int32_t cur = slot[h];
        if (cur < 0) return -1;
        int32_t o[3];
        fkey(facets, cur, o);
        if (o[0] == k[0] && o[1] == k[1] && o[2] == k[2]) return cur;
        h = (h + 1) & mask;
    }
}
__global__ void k_facet_match(int64_t E, const int32_t* tets, const uint8_t* on, const int32_t* facets,
                              const int32_t* slot, uint64_t mask, int32_t* cnt, int32_t* own) {
    GRID_STRIDE(e, E) {
        const int4 t4 = ((const int4*)tets)[e];
        const int32_t t[4] = {t4.x, t4.y, t4.z, t4.w};
        if (on[t[0]] + on[t[1]] + on[t[2]] + on[t[3]] < 3) continue;
        const int tf[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
        for (int j = 0; j < 4; ++j) {
            if (!on[t[tf[j][0]]] || !on[t[tf[j][1]]] || !on[t[tf[j][2]]]) continue;
            int32_t k[3] = {t[tf[j][0]], t[tf[j][1]], t[tf[j][2]]};
            sort3d(k);
            const int32_t g = facet_find(facets, slot, mask, k);
            if (g < 0) continue;
            atomicAdd(&cnt[g], 1);
            atomicMin(&own[g], (int32_t)e);
        }
    }
}
__global__ void k_facet_owner(int64_t F, const int32_t* facets, const int32_t* slot, uint64_t mask, const int32_t* cnt,
                              const int32_t* own, int32_t* owner, FinFlags* fl) {
    GRID_STRIDE(f, F) {
        int32_t k[3];
        fkey(facets, (int32_t)f, k);
        const int32_t g = facet_find(facets, slot, mask, k);
        if (g < 0 || cnt[g] != 1) fl->facet_error = 1;
        else owner[f] = own[g];
    }
}

// finalize over the device arrays already in m (tets unoriented); true when the mesh passed
bool finalize_device(DevMesh& m, cudaStream_t s) {
    DBuf T;
    FinFlags* f = T.alloc<FinFlags>(1);
    FinFlags h0{};
    h0.bad_elem = ~0ull;
    h0.max_region = -1;
    for (auto& v : h0.region_min_edge) v = 0x7ff0000000000000ull;  // +inf
    h2d(f, &h0, 1, s);
    const int64_t N = m.N, E = m.E, F = m.F;
    if (N) k_check_coords<<<grid_of(3 * N), 256, 0, s>>>(3 * N, m.coords, f);
    if (E) k_orient<<<grid_of(E), 256, 0, s>>>(E, m.N, m.tets, m.region, m.coords, f);
    DP_CHECK(cudaGetLastError());
    FinFlags h = read1(f, s);
    if (h.bad_coord || h.bad_elem != ~0ull) return false;
    m.node_region = m.mem.alloc<int32_t>(N);
    DP_CHECK(cudaMemsetAsync(m.node_region, 0xff, N * sizeof(int32_t), s));
    if (E) k_node_region<<<grid_of(4 * E), 256, 0, s>>>(E, m.tets, m.region, m.node_region, f);
    if (N) k_unreferenced<<<grid_of(N), 256, 0, s>>>(N, m.node_region, f);
    DP_CHECK(cudaGetLastError());
    h = read1(f, s);
    if (h.region_conflict || h.unreferenced) return false;
    m.h_owner.assign(F, -1);
    if (F) {
        uint8_t* on = T.alloc<uint8_t>(N);
        DP_CHECK(cudaMemsetAsync(on, 0, N, s));
        k_facet_nodes<<<grid_of(3 * F), 256, 0, s>>>(F, m.N, m.facets, on, f);
        h = read1(f, s);
        if (h.bad_facet_node) return false;
        size_t cap = 16;
        while (cap < 2 * (size_t)F + 16) cap <<= 1;
        int32_t* slot = T.alloc<int32_t>(cap);
        DP_CHECK(cudaMemsetAsync(slot, 0xff, cap * sizeof(int32_t), s));
        k_facet_insert<<<grid_of(F), 256, 0, s>>>(F, m.facets, slot, cap - 1);
        int32_t* cnt = T.alloc<int32_t>(F);
        int32_t* own = T.alloc<int32_t>(F);
        DP_CHECK(cudaMemsetAsync(cnt, 0, F * sizeof(int32_t), s));
        DP_CHECK(cudaMemsetAsync(own, 0x7f, F * sizeof(int32_t), s));
        k_facet_match<<<grid_of(E), 256, 0, s>>>(E, m.tets, on, m.facets, slot, cap - 1, cnt, own);
        int32_t* owner = T.alloc<int32_t>(F);
        k_facet_owner<<<grid_of(F), 256, 0, s>>>(F, m.facets, slot, cap - 1, cnt, own, owner, f);
        DP_CHECK(cudaGetLastError());
        h = read1(f, s);
        if (h.facet_error) return false;
        d2h(m.h_owner.data(), owner, F, s);
    }
    for (size_t c = 0; c < m.contacts.size(); ++c)
        if (m.contacts[c] < 0 || m.contacts[c] >= (int32_t)m.tags.size()) return false;
    m.max_region = h.max_region;
    m.region_count = h.max_region + 1;
    m.region_mask = h.region_mask;
    m.region_min_edge.assign(std::max(0, m.region_count), INFINITY);
    for (int r = 0; r < std::min(32, m.region_count); ++r) {
        const unsigned long long b = h.region_min_edge[r];
        double v;
        std::memcpy(&v, &b, 8);
        m.region_min_edge[r] = v;
    }
    // regions >= 32 are not tracked here: any region without a material (n_materials <= 16) is
    // reported by the setup resolution, as on the host
    return true;
}

// ------------------------------------------------------------------ fixture (generate_fixture)
__host__ __device__ __forceinline__ uint64_t splitmix_d(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double counter_uniform_d(uint64_t seed, uint64_t key) {
    const uint64_t z = splitmix_d(seed * 0x9E3779B97F4A7C15ull + splitmix_d(key + 0x632BE59BD9B4E019ull));
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

struct FixSpec {
    int kind, n;
    bool exact;
    int64_t r100;
    double radius, jitter, h;
    uint64_t seed;
};
__device__ __forceinline__ int32_t fx_cell_region(const FixSpec& s, int64_t i, int64_t j, int64_t k) {
    if (s.kind == 0) return 0;
    const int64_t n = s.n;
    const int64_t a = 2 * i + 1 - n, b = 2 * j + 1 - n, c = 2 * k + 1 - n;
    const int64_t q = a * a + b * b + c * c;
    const bool cast = s.exact ? (100 * q <= 4 * s.r100 * n * n) : ((double)q <= 4.0 * s.radius * s.radius * (double)n * n);
    return cast ? 0 : 1;
}
__device__ __forceinline__ int32_t fx_nb_region(const FixSpec& s, int64_t i, int64_t j, int64_t k) {
    if (i < 0 || j < 0 || k < 0 || i >= s.n || j >= s.n || k >= s.n) return -1;
    return fx_cell_region(s, i, j, k);
}
// regions touching grid point (i, j, k): bit r
__device__ __forceinline__ uint32_t fx_touch(const FixSpec& s, int64_t i, int64_t j, int64_t k) {
    uint32_t t = 0;
    for (int d = 0; d < 8; ++d) {
        const int64_t ci = i - (d & 1), cj = j - ((d >> 1) & 1), ck = k - ((d >> 2) & 1);
        const int32_t r = fx_nb_region(s, ci, cj, ck);
        if (r >= 0) t |= 1u << r;
    }
    return t;
}
__global__ void k_fx_touch(FixSpec s, int64_t G, int32_t* cnt) {
    const int64_t P = s.n + 1;
    GRID_STRIDE(g, G) cnt[g] = __popc(fx_touch(s, g % P, (g / P) % P, g / (P * P)));
}
__device__ __forceinline__ int32_t fx_node(const FixSpec& s, const int32_t* first, int64_t i, int64_t j, int64_t k,
                                           int32_t reg) {
    const int64_t P = s.n + 1;
    const int64_t g = i + P * (j + P * k);
    return first[g] + ((reg == 1 && (fx_touch(s, i, j, k) & 1)) ? 1 : 0);
}
__global__ void k_fx_coords(FixSpec s, int64_t G, const int32_t* first, double* X, int32_t* grid) {
    const int64_t P = s.n + 1;
    GRID_STRIDE(g, G) {
        const int64_t i = g % P, j = (g / P) % P, k = g / (P * P);
        double x[3] = {i * s.h, j * s.h, k * s.h};
        const int64_t gi[3] = {i, j, k};
        if (s.jitter != 0 && i > 0 && j > 0 && k > 0 && i < s.n && j < s.n && k < s.n)
            for (int d = 0; d < 3; ++d)
                x[d] = (double)gi[d] * s.h + (2.0 * counter_uniform_d(s.seed, 3 * (uint64_t)g + d) - 1.0) * s.jitter * s.h;
        for (int64_t id = first[g]; id < first[g + 1]; ++id) {
            for (int d = 0; d < 3; ++d) X[3 * id + d] = x[d];
            grid[id] = (int32_t)g;
        }
    }
}
__constant__ int c_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
__global__ void k_fx_fcount(FixSpec s, int64_t C, int32_t* fc) {
    const int64_t n = s.n;
    GRID_STRIDE(c, C) {
        const int64_t i = c % n, j = (c / n) % n, k = c / (n * n);
        const int32_t rg = fx_cell_region(s, i, j, k);
        int cnt = 0;
        for (int t = 0; t < 6; ++t) {
            const int a = c_perm[t][0], cc = c_perm[t][2];
            int64_t lo[3] = {i, j, k}, hi[3] = {i, j, k};
            lo[cc] -= 1;
            hi[a] += 1;
            cnt += fx_nb_region(s, lo[0], lo[1], lo[2]) != rg;
            cnt += fx_nb_region(s, hi[0], hi[1], hi[2]) != rg;
        }
        fc[c] = cnt;
    }
}
__global__ void k_fx_cells(FixSpec s, int64_t C, const int32_t* first, const int32_t* foff, int32_t* tets, int32_t* region,
                           int32_t* facets, int32_t* ftag) {
    const int64_t n = s.n;
    GRID_STRIDE(c, C) {
        const int64_t i = c % n, j = (c / n) % n, k = c / (n * n);
        const int32_t rg = fx_cell_region(s, i, j, k);
        int64_t fi = foff[c];
        for (int t = 0; t < 6; ++t) {
            const int a = c_perm[t][0], b = c_perm[t][1], cc = c_perm[t][2];
            int64_t v[4][3] = {{i, j, k}, {i, j, k}, {i, j, k}, {i + 1, j + 1, k + 1}};
            v[1][a] += 1;
            v[2][a] += 1;
            v[2][b] += 1;
            const int64_t e = 6 * c + t;
            for (int q = 0; q < 4; ++q) tets[4 * e + q] = fx_node(s, first, v[q][0], v[q][1], v[q][2], rg);
            region[e] = rg;
            int64_t lo[3] = {i, j, k}, hi[3] = {i, j, k};
            lo[cc] -= 1;
            hi[a] += 1;
            const int32_t nr[2] = {fx_nb_region(s, lo[0], lo[1], lo[2]), fx_nb_region(s, hi[0], hi[1], hi[2])};
            const int faces[2][3] = {{0, 1, 2}, {1, 2, 3}};
            for (int sd = 0; sd < 2; ++sd) {
                if (nr[sd] == rg) continue;
                for (int q = 0; q < 3; ++q) {
                    const int64_t* p = v[faces[sd][q]];
                    facets[3 * fi + q] = fx_node(s, first, p[0], p[1], p[2], rg);
                }
                ftag[fi] = nr[sd] < 0 ? 0 : (rg == 0 ? 1 : 2);
                ++fi;
            }
        }
    }
}

}  // namespace

void devmesh_from_desc(const cf_mesh_desc* d, cudaStream_t s, DevMesh& m) {
    if (!d || d->n_nodes < 0 || d->n_elems < 0 || d->n_facets < 0) raise(CF_INVALID_ARG, "bad mesh descriptor");
    if ((d->n_nodes && !d->coords) || (d->n_elems && (!d->tets || !d->region)) ||
        (d->n_facets && (!d->facets || !d->facet_tag)) || (d->n_tags && !d->tags) || (d->n_contacts && !d->contacts))
        raise(CF_INVALID_ARG, "null array in mesh descriptor");
    m.N = d->n_nodes;
    m.E = d->n_elems;
    m.F = d->n_facets;
    m.coords = m.mem.alloc<double>(3 * (size_t)m.N);
    m.tets = m.mem.alloc<int32_t>(4 * (size_t)m.E);
    m.region = m.mem.alloc<int32_t>(m.E);
    m.facets = m.mem.alloc<int32_t>(3 * (size_t)m.F);
    h2d(m.coords, d->coords, 3 * (size_t)m.N, s);
    h2d(m.tets, d->tets, 4 * (size_t)m.E, s);
    h2d(m.region, d->region, m.E, s);
    h2d(m.facets, d->facets, 3 * (size_t)m.F, s);
    m.h_facets.assign(d->facets, d->facets + 3 * (size_t)m.F);
    m.h_facet_tag.assign(d->facet_tag, d->facet_tag + m.F);
    m.tags.clear();
    for (int32_t t = 0; t < d->n_tags; ++t) m.tags.emplace_back(d->tags[t] ? d->tags[t] : "");
    m.contacts.assign(d->contacts, d->contacts + 2 * (size_t)d->n_contacts);
    for (int32_t f = 0; f < m.F; ++f)
        if (m.h_facet_tag[f] < 0 || m.h_facet_tag[f] >= (int32_t)m.tags.size())
            raise(CF_VALIDATION, "facet " + std::to_string(f) + " has an unknown tag");
    if (!finalize_device(m, s)) {
        MeshData hm;  // the host finalize raises the reference's message for the first defect
        finalize_mesh(d, hm);
        raise(CF_VALIDATION, "mesh validation failed on the device");
    }
}

namespace {
// permute_mesh reorder.hpp:152-163: node p moves to new_of_old[p]
__global__ void k_permute_nodes(int64_t N, const int32_t* p, const double* X, const int32_t* grid, double* X2,
                                int32_t* grid2) {
    GRID_STRIDE(n, N) {
        const int64_t q = p[n];
        X2[3 * q] = X[3 * n];
        X2[3 * q + 1] = X[3 * n + 1];
        X2[3 * q + 2] = X[3 * n + 2];
        if (grid) grid2[q] = grid[n];
    }
}
__global__ void k_relabel(int64_t n, const int32_t* p, int32_t* ids) {
    GRID_STRIDE(i, n) ids[i] = p[ids[i]];
}
}  // namespace

void devmesh_fixture(int kind, int n, double radius, double jitter, uint64_t seed, bool rcm, cudaStream_t s,
                     DevMesh& m) {
    if (n < 1 || n > 1024) raise(CF_INVALID_ARG, "fixture n out of range [1, 1024]");
    if (kind != 0 && kind != 1) raise(CF_INVALID_ARG, "fixture kind must be 0 (cube) or 1 (casting)");
    FixSpec sp{};
    sp.kind = kind;
    sp.n = n;
    sp.radius = radius;
    sp.jitter = jitter;
    sp.seed = seed;
    sp.h = 1.0 / n;
    sp.r100 = (int64_t)std::llround(radius * radius * 100.0);
    sp.exact = std::fabs(radius * radius * 100.0 - (double)sp.r100) < 1e-9;
    const int64_t P = n + 1, G = P * P * P, C = (int64_t)n * n * n, E = 6 * C;
    DBuf T;
    int32_t* cnt = T.alloc<int32_t>(G);
    k_fx_touch<<<grid_of(G), 256, 0, s>>>(sp, G, cnt);
    int32_t* first = T.alloc<int32_t>(G + 1);
    excl_sum(cnt, first, G, s);
    T.free(cnt);
    const int32_t N = read1(first + G, s);
    int32_t* fc = T.alloc<int32_t>(C);
    k_fx_fcount<<<grid_of(C), 256, 0, s>>>(sp, C, fc);
    int32_t* foff = T.alloc<int32_t>(C + 1);
    excl_sum(fc, foff, C, s);
    T.free(fc);
    const int32_t F = read1(foff + C, s);
    if (E > INT32_MAX) raise(CF_INVALID_ARG, "fixture too large for int32 ids");
    m.N = N;
    m.E = (int32_t)E;
    m.F = F;
    m.coords = m.mem.alloc<double>(3 * (size_t)N);
    m.node_grid = m.mem.alloc<int32_t>(N);
    m.tets = m.mem.alloc<int32_t>(4 * (size_t)E);
    m.region = m.mem.alloc<int32_t>(E);
    m.facets = m.mem.alloc<int32_t>(3 * (size_t)F);
    int32_t* ftag = T.alloc<int32_t>(F);
    k_fx_coords<<<grid_of(G), 256, 0, s>>>(sp, G, first, m.coords, m.node_grid);
    k_fx_cells<<<grid_of(C, 128), 128, 0, s>>>(sp, C, first, foff, m.tets, m.region, m.facets, ftag);
    DP_CHECK(cudaGetLastError());
    if (rcm) {  // the generated mesh renumbered by rcm_permutation (the reference's preprocessing)
        DBuf P;
        int32_t* lab = P.alloc<int32_t>(N);
        rcm_labels_device(N, E, m.tets, -1, s, lab);
        double* X2 = m.mem.alloc<double>(3 * (size_t)N);
        int32_t* g2 = m.mem.alloc<int32_t>(N);
        k_permute_nodes<<<grid_of(N), 256, 0, s>>>(N, lab, m.coords, m.node_grid, X2, g2);
        k_relabel<<<grid_of(4 * E), 256, 0, s>>>(4 * E, lab, m.tets);
        if (F) k_relabel<<<grid_of(3 * (int64_t)F), 256, 0, s>>>(3 * (int64_t)F, lab, m.facets);
        DP_CHECK(cudaGetLastError());
        DP_CHECK(cudaStreamSynchronize(s));
        m.mem.free(m.coords);
        m.mem.free(m.node_grid);
        m.coords = X2;
        m.node_grid = g2;
    }
    m.h_facets.resize(3 * (size_t)F);
    m.h_facet_tag.resize(F);
    d2h(m.h_facets.data(), m.facets, 3 * (size_t)F, s);
    d2h(m.h_facet_tag.data(), ftag, F, s);
    m.tags = kind == 1 ? std::vector<std::string>{"outer", "cast_if", "mold_if"} : std::vector<std::string>{"outer"};
    m.contacts = kind == 1 ? std::vector<int32_t>{1, 2} : std::vector<int32_t>{};
    if (!finalize_device(m, s)) raise(CF_VALIDATION, "generated fixture failed validation");
}

// ------------------------------------------------------------------ setup resolution
namespace {
__global__ void k_first_bad_region(int64_t E, const int32_t* region, int32_t nmat, unsigned long long* first) {
    GRID_STRIDE(e, E) if (region[e] >= nmat) atomicMin(first, (unsigned long long)e);
}
__global__ void k_gather3(int64_t n, const int32_t* ids, const double* X, double* out) {
    GRID_STRIDE(i, n) {
        const int64_t v = ids[i];
        out[3 * i] = X[3 * v];
        out[3 * i + 1] = X[3 * v + 1];
        out[3 * i + 2] = X[3 * v + 2];
    }
}
__global__ void k_dir_best(int64_t nf, const int32_t* flist, const int32_t* facets, const int32_t* ftag, int32_t* best) {
    GRID_STRIDE(i, nf) {
        const int32_t f = flist[i];
        for (int a = 0; a < 3; ++a) atomicMin(&best[facets[3 * (int64_t)f + a]], ftag[f]);
    }
}
__global__ void k_dir_final(int64_t N, const int32_t* best, const int32_t* kind_of_tag, int32_t* dir) {
    GRID_STRIDE(n, N) dir[n] = best[n] == INT32_MAX ? -1 : -1 - kind_of_tag[best[n]];
}
struct T0Args {
    double mat_T0[kMaxRegions];
    double dir_T0[kMaxFacetKinds];
    double amp;
    uint64_t seed;
};
__global__ void k_T0(int64_t N, const int32_t* nreg, const int32_t* dir, const double* init, const int32_t* grid,
                     T0Args a, double* T0) {
    GRID_STRIDE(n, N) {
        double v;
        if (init) {
            v = init[n];
        } else {
            v = a.mat_T0[nreg[n]];
            if (a.amp != 0) v = v + (-a.amp + (a.amp - -a.amp) * counter_uniform_d(a.seed, (uint64_t)grid[n]));
        }
        if (dir && dir[n] >= 0) v = a.dir_T0[dir[n]];
        T0[n] = v;
    }
}
}  // namespace

void resolve_setup_device(const DevMesh& m, const cf_setup_desc* s, const T0Noise& noise, cudaStream_t st,
                          DevSetup& out) {
    if (!s) raise(CF_INVALID_ARG, "null setup");
    // the facet part of the mesh on the host: facets over the compacted set of facet nodes
    MeshData fm;
    std::vector<int32_t> fnodes(m.h_facets);
    std::sort(fnodes.begin(), fnodes.end());
    fnodes.erase(std::unique(fnodes.begin(), fnodes.end()), fnodes.end());
    std::vector<int32_t> cfacets(m.h_facets.size());
    for (size_t i = 0; i < cfacets.size(); ++i)
        cfacets[i] = (int32_t)(std::lower_bound(fnodes.begin(), fnodes.end(), m.h_facets[i]) - fnodes.begin());
    std::vector<double> fcoords(3 * fnodes.size());
    if (!fnodes.empty()) {
        DBuf T;
        int32_t* ids = T.alloc<int32_t>(fnodes.size());
        double* xo = T.alloc<double>(3 * fnodes.size());
        h2d(ids, fnodes.data(), fnodes.size(), st);
        k_gather3<<<grid_of((int64_t)fnodes.size()), 256, 0, st>>>((int64_t)fnodes.size(), ids, m.coords, xo);
        d2h(fcoords.data(), xo, fcoords.size(), st);
    }
    fm.N = (int32_t)fnodes.size();
    fm.E = 0;
    fm.F = m.F;
    fm.coords = fcoords.data();
    fm.facets = cfacets.data();
    fm.facet_tag = m.h_facet_tag.data();
    fm.owner = m.h_owner;
    fm.tags = m.tags;
    fm.contacts = m.contacts;
    fm.region_count = m.region_count;
    fm.region_min_edge = m.region_min_edge;
    RegionUse ru;
    ru.mask = m.region_mask;
    {
        DBuf T;
        unsigned long long* first = T.alloc<unsigned long long>(1);
        const unsigned long long init = ~0ull;
        h2d(first, &init, 1, st);
        if (m.E) k_first_bad_region<<<grid_of(m.E), 256, 0, st>>>(m.E, m.region, s->n_materials, first);
        const unsigned long long e = read1(first, st);
        if (e != ~0ull) ru.first_bad_region = read1(m.region + e, st);
    }
    resolve_setup_impl(fm, s, out.S, &ru, false);
    SetupData& S = out.S;
    // Dirichlet nodes (lowest tag wins, blocked.hpp:250-263) and T0 (initial_temperatures :396-417)
    std::vector<int32_t> dfac;
    for (int32_t f = 0; f < m.F; ++f)
        if (S.facet_kind[f] < 0) dfac.push_back(f);
    const int64_t N = m.N;
    if (!dfac.empty()) {
        DBuf T;
        int32_t* fl = T.alloc<int32_t>(dfac.size());
        int32_t* ftag = T.alloc<int32_t>(m.F);
        int32_t* best = T.alloc<int32_t>(N);
        int32_t* kot = T.alloc<int32_t>(S.kind_of_tag.size());
        h2d(fl, dfac.data(), dfac.size(), st);
        h2d(ftag, m.h_facet_tag.data(), m.F, st);
        h2d(kot, S.kind_of_tag.data(), S.kind_of_tag.size(), st);
        k_fill<<<grid_of(N), 256, 0, st>>>(N, best, INT32_MAX);
        k_dir_best<<<grid_of((int64_t)dfac.size()), 256, 0, st>>>((int64_t)dfac.size(), fl, m.facets, ftag, best);
        out.dir_of_node = out.mem.alloc<int32_t>(N);
        k_dir_final<<<grid_of(N), 256, 0, st>>>(N, best, kot, out.dir_of_node);
        DP_CHECK(cudaGetLastError());
        DP_CHECK(cudaStreamSynchronize(st));
    }
    T0Args a{};
    for (int r = 0; r < s->n_materials && r < kMaxRegions; ++r) a.mat_T0[r] = s->materials[r].initial_temperature;
    for (int d = 0; d < kMaxFacetKinds; ++d)
        if (S.P.dir_tab[d].n > 0) a.dir_T0[d] = pl_eval(S.P, S.P.dir_tab[d], 0.0);
    a.amp = s->initial_T ? 0.0 : noise.amp;
    a.seed = noise.seed;
    if (a.amp != 0 && !m.node_grid) raise(CF_INVALID_ARG, "T0 noise needs a generated fixture (node grid)");
    out.T0 = out.mem.alloc<double>(N);
    DBuf T;
    double* init = nullptr;
    if (s->initial_T) {
        init = T.alloc<double>(N);
        h2d(init, s->initial_T, N, st);
    }
    if (N) k_T0<<<grid_of(N), 256, 0, st>>>(N, m.node_region, out.dir_of_node, init, m.node_grid, a, out.T0);
    DP_CHECK(cudaGetLastError());
    DP_CHECK(cudaStreamSynchronize(st));
}

// ------------------------------------------------------------------ RCB on the device
namespace {
__device__ __forceinline__ double centroid_rcb(const int32_t* tets, const double* X, int32_t e, int k) {
    const int4 t = ((const int4*)tets)[e];
    return (((X[3 * (int64_t)t.x + k] + X[3 * (int64_t)t.y + k]) + X[3 * (int64_t)t.z + k]) + X[3 * (int64_t)t.w + k]) * 0.25;
}
__global__ void k_rcb_bbox(int64_t n, const int32_t* ids, const int32_t* tets, const double* X, unsigned long long* bb) {
    GRID_STRIDE(i, n) {
        for (int k = 0; k < 3; ++k) {
            const unsigned long long v = dkey(centroid_rcb(tets, X, ids[i], k));
            atomicMin(&bb[k], v);
            atomicMax(&bb[3 + k], v);
        }
    }
}
__global__ void k_rcb_keys(int64_t n, const int32_t* ids, const int32_t* tets, const double* X, int axis, uint64_t* key) {
    GRID_STRIDE(i, n) key[i] = dkey(centroid_rcb(tets, X, ids[i], axis));
}
__global__ void k_iota(int64_t n, int32_t* a) {
    GRID_STRIDE(i, n) a[i] = (int32_t)i;
}
__global__ void k_set_part(int64_t n, const int32_t* ids, int32_t v, int32_t* part) {
    GRID_STRIDE(i, n) part[ids[i]] = v;
}
}  // namespace

void partition_rcb_device(const DevMesh& m, int32_t parts, cudaStream_t s, int32_t* part) {
    if (parts < 1) raise(CF_INVALID_ARG, "parts must be >= 1");
    const int64_t E = m.E;
    DBuf T;
    int32_t* ids = T.alloc<int32_t>(E);
    int32_t* ids2 = T.alloc<int32_t>(E);
    uint64_t* key = T.alloc<uint64_t>(E);
    uint64_t* key2 = T.alloc<uint64_t>(E);
    unsigned long long* bb = T.alloc<unsigned long long>(6);
    if (E) k_iota<<<grid_of(E), 256, 0, s>>>(E, ids);
    struct Job {
        int64_t lo, hi;
        int32_t first, count;
    };
    std::vector<Job> stack{{0, E, 0, parts}};
    while (!stack.empty()) {
        const Job j = stack.back();
        stack.pop_back();
        const int64_t n = j.hi - j.lo;
        if (j.count == 1) {
            if (n) k_set_part<<<grid_of(n), 256, 0, s>>>(n, ids + j.lo, j.first, part);
            continue;
        }
        unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
        h2d(bb, init, 6, s);
        if (n) k_rcb_bbox<<<grid_of(n), 256, 0, s>>>(n, ids + j.lo, m.tets, m.coords, bb);
        unsigned long long h[6];
        d2h(h, bb, 6, s);
        double lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
            lo[k] = n ? dval(h[k]) : INFINITY;
            hi[k] = n ? dval(h[3 + k]) : -INFINITY;
        }
        int axis = 0;
        for (int k = 1; k < 3; ++k)
            if (hi[k] - lo[k] > hi[axis] - lo[axis]) axis = k;
        const int32_t left = j.count / 2;
        const int64_t nl = n * left / j.count;
        // the nl smallest by (coordinate, id): ids ascending, then a stable sort by coordinate
        if (n > 1) {
            sort_keys(ids + j.lo, ids2 + j.lo, n, 32, s);
            k_rcb_keys<<<grid_of(n), 256, 0, s>>>(n, ids2 + j.lo, m.tets, m.coords, axis, key);
            sort_pairs(key, key2, ids2 + j.lo, ids + j.lo, n, 64, s);
        }
        stack.push_back({j.lo + nl, j.hi, j.first + left, j.count - left});
        stack.push_back({j.lo, j.lo + nl, j.first, left});
    }
    DP_CHECK(cudaGetLastError());
    DP_CHECK(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ tile builder
namespace {
__global__ void k_bbox_nodes(int64_t N, const double* X, unsigned long long* bb) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    GRID_STRIDE(n, N) {
        for (int k = 0; k < 3; ++k) {
            const unsigned long long v = dkey(X[3 * n + k]);
            lo[k] = v < lo[k] ? v : lo[k];
            hi[k] = v > hi[k] ? v : hi[k];
        }
    }
    for (int k = 0; k < 3; ++k) {
        atomicMin(&bb[k], lo[k]);
        atomicMax(&bb[3 + k], hi[k]);
    }
}
__device__ __forceinline__ uint64_t spread21d(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}
struct Box {
    double lo[3], span;
};
// Morton code of the element centroid (the host's operation order, cf_plan.cpp)
__global__ void k_morton(int64_t n, const int32_t* elems, const int32_t* tets, const double* X, Box b, uint64_t* key,
                         int32_t* val) {
    GRID_STRIDE(i, n) {
        const int32_t e = elems ? elems[i] : (int32_t)i;
        const int4 t = ((const int4*)tets)[e];
        uint64_t code = 0;
        for (int k = 0; k < 3; ++k) {
            const double c = 0.25 * (X[3 * (int64_t)t.x + k] + X[3 * (int64_t)t.y + k] + X[3 * (int64_t)t.z + k] +
                                     X[3 * (int64_t)t.w + k]);
            double q = (c - b.lo[k]) / b.span * 2097151.0;
            q = q < 0.0 ? 0.0 : q;
            q = 2097151.0 < q ? 2097151.0 : q;
            code |= spread21d((uint64_t)q) << k;
        }
        key[i] = code;
        val[i] = e;
    }
}
__global__ void k_minnode(int64_t n, const int32_t* elems, const int32_t* tets, const int32_t* label, uint32_t* key,
                          int32_t* val) {
    GRID_STRIDE(i, n) {
        const int32_t e = elems ? elems[i] : (int32_t)i;
        const int4 t = ((const int4*)tets)[e];
        const int32_t q[4] = {t.x, t.y, t.z, t.w};
        int32_t mn = INT32_MAX;
        for (int a = 0; a < 4; ++a) {
            const int32_t l = label ? label[q[a]] : q[a];
            mn = l < mn ? l : mn;
        }
        key[i] = (uint32_t)mn;
        val[i] = e;
    }
}
__global__ void k_footprint(TileCtx c, const int32_t* order, const int64_t* rs, const int32_t* rl, int64_t nr,
                            int32_t* ws, int64_t ws_ints, int64_t* fp) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nr) return;
    fp[i] = tile_footprint(c, order + rs[i], rl[i], ws + i * ws_ints);
}
__global__ void k_mark(int64_t n, const int32_t* elems, const int32_t* tets, uint8_t* mark) {
    GRID_STRIDE(k, 4 * n) mark[tets[4 * (int64_t)elems[k >> 2] + (k & 3)]] = 1;
}
__global__ void k_first_touch(int64_t n, const int32_t* order, const int32_t* tets, unsigned long long* ft) {
    GRID_STRIDE(k, 4 * n) atomicMin(&ft[tets[4 * (int64_t)order[k >> 2] + (k & 3)]], (unsigned long long)k);
}
__global__ void k_inv(int64_t N, const int32_t* label, int32_t* inv) {
    GRID_STRIDE(n, N) inv[label ? label[n] : n] = (int32_t)n;
}
__global__ void k_flag_by_label(int64_t N, const int32_t* inv, const uint8_t* mark, int32_t* flag) {
    GRID_STRIDE(l, N) flag[l] = mark ? mark[inv[l]] : 1;
}
__global__ void k_number_by_label(int64_t N, const int32_t* inv, const int32_t* flag, const int32_t* pos,
                                  int32_t* lnodes, int32_t* local_of) {
    GRID_STRIDE(l, N) {
        const int32_t n = inv[l];
        if (flag[l]) {
            lnodes[pos[l]] = n;
            local_of[n] = pos[l];
        } else {
            local_of[n] = -1;
        }
    }
}
__global__ void k_number_list(int64_t nl, const int32_t* lnodes, int32_t* local_of) {
    GRID_STRIDE(l, nl) local_of[lnodes[l]] = (int32_t)l;
}
__global__ void k_lnode_attr(int64_t nl, const int32_t* lnodes, const int32_t* nreg, const int32_t* dir, uint8_t* lreg,
                             int8_t* ldir, int32_t* any_dir) {
    GRID_STRIDE(l, nl) {
        const int32_t n = lnodes[l];
        lreg[l] = (uint8_t)nreg[n];
        if (dir) {
            const int32_t d = dir[n];
            if (ldir) ldir[l] = (int8_t)d;
            if (d >= 0) *any_dir = 1;
        }
    }
}
__global__ void k_pass1(TileCtx c, const int32_t* order, const int64_t* tstart, int64_t t0, int64_t t1, int32_t* ws,
                        int64_t ws_ints, TileMeta* meta, const int32_t* tn_off, int32_t* tnodes) {
    const int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= t1) return;
    const int ne = (int)(tstart[t + 1] - tstart[t]);
    int32_t* w = ws + (t - t0) * ws_ints;
    int32_t* tn = w;  // [4 ne] scratch for the ordered nodes
    const TileMeta tm = tile_pass1(c, order + tstart[t], ne, tn, w + 4 * ne);
    if (!tn_off) {
        meta[t] = tm;
    } else {
        int32_t* dst = tnodes + tn_off[t];
        for (int k = 0; k < tm.ns; ++k) dst[k] = tn[k];
    }
}
__global__ void k_ntiles(int64_t nt, const int32_t* tn_off, const int32_t* tnodes, int32_t* ntiles_of) {
    GRID_STRIDE(t, nt) for (int32_t k = tn_off[t]; k < tn_off[t + 1]; ++k) atomicAdd(&ntiles_of[tnodes[k]], 1);
}
__global__ void k_shared_node(int64_t nl, const int32_t* lnodes, const unsigned long long* nmask, uint8_t* shared) {
    GRID_STRIDE(l, nl) shared[l] = __popcll(nmask[lnodes[l]]) > 1;
}
__global__ void k_border(int64_t nt, const int32_t* tn_off, const int32_t* tnodes, const uint8_t* shared, uint8_t* border) {
    GRID_STRIDE(t, nt) {
        uint8_t b = 0;
        for (int32_t k = tn_off[t]; k < tn_off[t + 1]; ++k) b |= shared[tnodes[k]];
        border[t] = b;
    }
}
__global__ void k_nodemask(int64_t E, const int32_t* tets, const int32_t* part, unsigned long long* nmask) {
    GRID_STRIDE(k, 4 * E) {
        const unsigned long long bit = 1ull << part[k >> 2];
        unsigned long long* w = &nmask[tets[k]];
        if (!(*w & bit)) atomicOr(w, bit);
    }
}
__global__ void k_fe_count(int64_t nb, const int32_t* owner_of_bound, int32_t* cnt) {
    GRID_STRIDE(i, nb) atomicAdd(&cnt[owner_of_bound[i]], 1);
}
struct PackK {
    TileCtx c;
    const int32_t* order;
    const int64_t* tstart;
    const TileMeta* meta;
    const int32_t* tn_off;
    const int32_t* tnodes;
    const int64_t* blob_off;
    const int32_t* slot_off;
    uint8_t* blob;
    int32_t* slot_node;
    int32_t* elem_global;
    int32_t* ws;
    int64_t ws_ints;
    unsigned long long* counts;  // n_if, n_bc
};
__global__ void __launch_bounds__(128) k_pack(PackK a, int64_t t0, int64_t t1) {
    const int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= t1) return;
    const TileMeta tm = a.meta[t];
    const TileLayout L(tm, a.c.tdep, a.c.coords_layout);
    TileOut to;
    to.stg = a.blob + a.blob_off[t] + L.stage;
    to.elem_global = a.elem_global + a.tstart[t];
    to.tets_ord = nullptr;
    to.slot_node = a.slot_node + a.slot_off[t];
    tile_pack(a.c, (int32_t)t, a.order + a.tstart[t], tm, a.tnodes + a.tn_off[t], a.ws + (t - t0) * a.ws_ints, to);
    if (to.n_if) atomicAdd(&a.counts[0], (unsigned long long)to.n_if);
    if (to.n_bc) atomicAdd(&a.counts[1], (unsigned long long)to.n_bc);
}
// element geometry into the blob (fill_tiles_kernel's geometry part, over global node ids)
__global__ void __launch_bounds__(128) k_fill_geom(const TileMeta* meta, const int64_t* blob_off, const int64_t* tstart,
                                                   const int32_t* elem_global, const int32_t* tets, const double* X,
                                                   const int32_t* slot_off, const int32_t* slot_node,
                                                   const int32_t* local_global, uint8_t* blob, bool tdep, bool coords) {
    const int64_t t = blockIdx.x;
    const TileMeta tm = meta[t];
    const TileLayout L(tm, tdep, coords);
    uint8_t* B = blob + blob_off[t];
    const int S = L.ne2;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        double g[4][3], vol = 0, mn = 0, mx = 0;
        if (i < tm.ne) {
            const int4 q = ((const int4*)tets)[elem_global[tstart[t] + i]];
            const int32_t nn[4] = {q.x, q.y, q.z, q.w};
            double p[4][3];
            for (int a = 0; a < 4; ++a)
                for (int k = 0; k < 3; ++k) p[a][k] = X[3 * (int64_t)nn[a] + k];
            dev_tet_geometry(p, g, vol, mn, mx);
        } else {
            for (int a = 0; a < 4; ++a) g[a][0] = g[a][1] = g[a][2] = 0.0;
        }
        if (coords) {
            ((double*)(B + L.geom))[i] = mx;
        } else {
            double2* G2 = (double2*)(B + L.geom);
            G2[i] = make_double2(g[1][0], g[1][1]);
            G2[S + i] = make_double2(g[1][2], g[2][0]);
            G2[2 * S + i] = make_double2(g[2][1], g[2][2]);
            G2[3 * S + i] = make_double2(g[3][0], g[3][1]);
            G2[4 * S + i] = make_double2(g[3][2], vol);
            *(double*)(B + L.max_edge_of(i)) = mx;
        }
        if (tdep) ((double*)(B + L.minedge))[i] = mn;
    }
    if (coords) {
        double* xyz = (double*)(B + L.xyz);
        const int s0 = slot_off[t];
        for (int k = threadIdx.x; k < tm.ns; k += blockDim.x) {
            const int64_t n = local_global[slot_node[s0 + k] & 0x0fffffff];
            xyz[4 * k] = X[3 * n];
            xyz[4 * k + 1] = X[3 * n + 1];
            xyz[4 * k + 2] = X[3 * n + 2];
            xyz[4 * k + 3] = 0.0;
        }
    }
}
__global__ void k_merge_keys(int64_t S, const int32_t* slot_node, int32_t sentinel, int32_t* key, int32_t* val,
                             int32_t* cnt) {
    GRID_STRIDE(s, S) {
        const int32_t sn = slot_node[s];
        const int32_t l = sn >= 0 ? (int32_t)((uint32_t)sn & 0x0fffffffu) : sentinel;
        key[s] = l;
        val[s] = (int32_t)s;
        if (sn >= 0) atomicAdd(&cnt[l], 1);
    }
}
__global__ void k_zero_tail(int64_t from, int64_t to, int32_t* a) {
    for (int64_t i = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < to; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = 0;
}
__global__ void k_shared_keys(int64_t nl, const int32_t* ntiles_of, const uint8_t* shared, const int32_t* merge_off,
                              const int32_t* merge_idx, uint64_t* key, int32_t* val, unsigned long long* nsh) {
    GRID_STRIDE(l, nl) {
        const bool priv = ntiles_of[l] == 1 && !(shared && shared[l]);
        if (priv) {
            key[l] = ~0ull;
        } else {
            key[l] = merge_off[l + 1] > merge_off[l] ? (uint64_t)merge_idx[merge_off[l]] : (uint64_t)(INT64_MAX - nl + l);
            atomicAdd(nsh, 1ull);
        }
        val[l] = (int32_t)l;
    }
}
// update records (update_kernel): {node, count, slot0, slot1}, {slot2 .. slot5} + {slot6, slot7}
__global__ void k_shared_rec(int64_t n, const int32_t* list, const int32_t* merge_off, const int32_t* merge_idx,
                             int4* rec, int2* rec2, unsigned long long* parts) {
    GRID_STRIDE(k, n) {
        const int32_t i = list[k];
        const int32_t b = merge_off[i], cnt = merge_off[i + 1] - b;
        int32_t sl[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int q = 0; q < 8 && q < cnt; ++q) sl[q] = merge_idx[b + q];
        rec[2 * k] = make_int4(i, cnt, sl[0], sl[1]);
        rec[2 * k + 1] = make_int4(sl[2], sl[3], sl[4], sl[5]);
        rec2[k] = make_int2(sl[6], sl[7]);
        atomicAdd(parts, (unsigned long long)cnt);
    }
}
__global__ void k_gather_i32(int64_t n, const int32_t* idx, const int32_t* src, int32_t* out) {
    GRID_STRIDE(i, n) out[i] = idx[i] >= 0 ? src[idx[i]] : -1;
}
__global__ void k_gather_corners(int64_t n, const int32_t* elems, const int32_t* tets, int32_t* out) {
    GRID_STRIDE(i, 4 * n) out[i] = tets[4 * (int64_t)elems[i >> 2] + (i & 3)];
}
__global__ void k_gather_u64(int64_t n, const int32_t* idx, const unsigned long long* src, unsigned long long* out) {
    GRID_STRIDE(i, n) out[i] = src[idx[i]];
}
__global__ void k_scatter_i32(int64_t n, const int32_t* idx, const int32_t* v, int32_t* dst) {
    GRID_STRIDE(i, n) dst[idx[i]] = v[i];
}
__global__ void k_select_shared(int64_t nl, const int32_t* lnodes, const uint8_t* shared, int32_t* out_g,
                                int32_t* out_l, unsigned long long* out_m, const unsigned long long* nmask,
                                unsigned long long* cnt) {
    GRID_STRIDE(l, nl) {
        if (!shared[l]) continue;
        const unsigned long long k = atomicAdd(cnt, 1ull);
        out_g[k] = lnodes[l];
        out_l[k] = (int32_t)l;
        out_m[k] = nmask[lnodes[l]];
    }
}

struct Pred {
    const int32_t* part;
    int32_t r;
    __device__ bool operator()(int32_t e) const { return part[e] == r; }
};
struct NotMax {
    __device__ int64_t operator()(unsigned long long v) const { return v != ~0ull; }
};

int64_t ws_batch(int64_t ws_ints, int64_t n) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const int64_t budget = std::min<int64_t>(8ll << 30, (int64_t)fr / 4);
    return std::max<int64_t>(1, std::min<int64_t>(n, budget / std::max<int64_t>(1, 4 * ws_ints)));
}
}  // namespace

void build_rank_plan_device(const DevMesh& m, const DevSetup& DS, const PlanOptions& o, const int32_t* d_label,
                            const int32_t* d_part, int32_t rank, cudaStream_t s, DevRankPlan& out) {
    const SetupData& S = DS.S;
    RankPlan& rp = out.H;
    rp = RankPlan{};
    rp.rank = rank;
    rp.coords = o.geometry == CF_GEOM_COORDS;
    const bool coords = rp.coords;
    const int32_t W = o.world_size;
    if (W > 64) raise(CF_INVALID_ARG, "device setup supports at most 64 ranks");
    const int64_t E = m.E, N = m.N, F = m.F;
    DBuf T;  // transients
    DBuf& M = out.mem;
    // ---- elements of this rank (ascending id) and the parts touching each node
    int32_t* elems = nullptr;
    int64_t Er = E;
    unsigned long long* nmask = nullptr;
    std::vector<int32_t> owner_part;  // [F] part of each facet's owner (multi-rank)
    if (W > 1) {
        elems = T.alloc<int32_t>(E);
        unsigned long long* nsel = T.alloc<unsigned long long>(1);
        {
            cub::CountingInputIterator<int32_t> it(0);
            size_t tb = 0;
            DP_CHECK(cub::DeviceSelect::If(nullptr, tb, it, elems, nsel, E, Pred{d_part, rank}, s));
            DBuf TT;
            void* tmp = TT.alloc<uint8_t>(tb);
            DP_CHECK(cub::DeviceSelect::If(tmp, tb, it, elems, nsel, E, Pred{d_part, rank}, s));
            Er = (int64_t)read1(nsel, s);
        }
        nmask = T.alloc<unsigned long long>(N);
        DP_CHECK(cudaMemsetAsync(nmask, 0, N * sizeof(unsigned long long), s));
        k_nodemask<<<grid_of(4 * E), 256, 0, s>>>(E, m.tets, d_part, nmask);
        owner_part.resize(F);
        if (F) {
            DBuf TT;
            int32_t* own = TT.alloc<int32_t>(F);
            int32_t* op = TT.alloc<int32_t>(F);
            h2d(own, m.h_owner.data(), F, s);
            k_gather_i32<<<grid_of(F), 256, 0, s>>>(F, own, d_part, op);
            d2h(owner_part.data(), op, F, s);
        }
    }
    auto in_rank_owner = [&](int32_t f) { return W == 1 || owner_part[f] == rank; };
    // ---- facet bindings per element (ascending facet id), Dirichlet facets excluded
    std::vector<int32_t> bound, bound_owner;
    for (int32_t f = 0; f < F; ++f)
        if (in_rank_owner(f) && S.facet_kind[f] >= 0) bound.push_back(f);
    std::stable_sort(bound.begin(), bound.end(), [&](int32_t a, int32_t b) { return m.h_owner[a] < m.h_owner[b]; });
    for (int32_t f : bound) bound_owner.push_back(m.h_owner[f]);
    int32_t* fe = T.alloc<int32_t>(bound.size());
    int32_t* fe_off = T.alloc<int32_t>(E + 1);
    {
        DBuf TT;
        int32_t* bo = TT.alloc<int32_t>(bound.size());
        int32_t* cnt = TT.alloc<int32_t>(E);
        h2d(fe, bound.data(), bound.size(), s);
        h2d(bo, bound_owner.data(), bound_owner.size(), s);
        DP_CHECK(cudaMemsetAsync(cnt, 0, E * sizeof(int32_t), s));
        if (!bound.empty()) k_fe_count<<<grid_of((int64_t)bound.size()), 256, 0, s>>>((int64_t)bound.size(), bo, cnt);
        excl_sum(cnt, fe_off, E, s);
    }
    std::vector<int32_t> sister(F, -1);
    for (const Pair& q : S.pairs) sister[q.facet] = q.sister;
    int32_t* d_sister = T.alloc<int32_t>(F);
    int32_t* d_fkind = T.alloc<int32_t>(F);
    uint8_t* d_kind_if = T.alloc<uint8_t>(kMaxFacetKinds);
    {
        uint8_t kif[kMaxFacetKinds];
        for (int k = 0; k < kMaxFacetKinds; ++k) kif[k] = (uint8_t)(S.P.kind[k].interface != 0);
        h2d(d_sister, sister.data(), F, s);
        h2d(d_fkind, S.facet_kind.data(), F, s);
        h2d(d_kind_if, kif, kMaxFacetKinds, s);
    }
    TileCtx c;
    c.tets = m.tets;
    c.region = m.region;
    c.facets = m.facets;
    c.coords = m.coords;
    c.fe_off = fe_off;
    c.fe = fe;
    c.facet_kind = d_fkind;
    c.facet_sister = d_sister;
    c.kind_interface = d_kind_if;
    c.tdep = S.temp_dep;
    c.coords_layout = coords;
    tile_env(c);

    // ---- element order and chunks
    int32_t* order = T.alloc<int32_t>(Er);
    if (o.elem_order == CF_ELEM_ORDER_MORTON || o.elem_order == CF_ELEM_ORDER_MIN_NODE) {
        DBuf TT;
        int32_t* v0 = TT.alloc<int32_t>(Er);
        if (o.elem_order == CF_ELEM_ORDER_MORTON) {
            unsigned long long* bb = TT.alloc<unsigned long long>(6);
            unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
            h2d(bb, init, 6, s);
            k_bbox_nodes<<<grid_of(N), 256, 0, s>>>(N, m.coords, bb);
            unsigned long long h[6];
            d2h(h, bb, 6, s);
            Box b;
            double hi[3];
            for (int k = 0; k < 3; ++k) {
                b.lo[k] = N ? dval(h[k]) : INFINITY;
                hi[k] = N ? dval(h[3 + k]) : -INFINITY;
            }
            b.span = std::max({hi[0] - b.lo[0], hi[1] - b.lo[1], hi[2] - b.lo[2], 1e-300});
            uint64_t* k0 = TT.alloc<uint64_t>(Er);
            uint64_t* k1 = TT.alloc<uint64_t>(Er);
            if (Er) k_morton<<<grid_of(Er), 256, 0, s>>>(Er, elems, m.tets, m.coords, b, k0, v0);
            sort_pairs(k0, k1, v0, order, Er, 63, s);
        } else {
            uint32_t* k0 = TT.alloc<uint32_t>(Er);
            uint32_t* k1 = TT.alloc<uint32_t>(Er);
            if (Er) k_minnode<<<grid_of(Er), 256, 0, s>>>(Er, elems, m.tets, d_label, k0, v0);
            sort_pairs(k0, k1, v0, order, Er, 32, s);
        }
    } else if (elems) {
        DP_CHECK(cudaMemcpyAsync(order, elems, Er * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    } else if (Er) {
        k_iota<<<grid_of(Er), 256, 0, s>>>(Er, order);
    }
    if (elems) T.free(elems);
    const int TE = o.tile_elems;
    std::vector<int64_t> rstart;
    std::vector<int32_t> rlen;
    for (int64_t i = 0; i < Er; i += TE) {
        rstart.push_back(i);
        rlen.push_back((int32_t)std::min<int64_t>(TE, Er - i));
    }
    // shared-memory budget: 95th percentile of the chunk footprints; larger chunks are halved
    // along the order until they fit (or hold <= 16 elements)
    auto footprints = [&](const std::vector<int64_t>& st, const std::vector<int32_t>& ln) {
        std::vector<int64_t> fp(st.size());
        if (st.empty()) return fp;
        int32_t mx = *std::max_element(ln.begin(), ln.end());
        const int64_t wsi = 8 * (int64_t)mx + 64;
        const int64_t batch = ws_batch(wsi, (int64_t)st.size());
        DBuf TT;
        int32_t* ws = TT.alloc<int32_t>(batch * wsi);
        int64_t* d_rs = TT.alloc<int64_t>(st.size());
        int32_t* d_rl = TT.alloc<int32_t>(st.size());
        int64_t* d_fp = TT.alloc<int64_t>(st.size());
        h2d(d_rs, st.data(), st.size(), s);
        h2d(d_rl, ln.data(), ln.size(), s);
        for (int64_t b0 = 0; b0 < (int64_t)st.size(); b0 += batch) {
            const int64_t nb = std::min<int64_t>(batch, (int64_t)st.size() - b0);
            k_footprint<<<(int)((nb + 127) / 128), 128, 0, s>>>(c, order, d_rs + b0, d_rl + b0, nb, ws, wsi, d_fp + b0);
            DP_CHECK(cudaGetLastError());
        }
        d2h(fp.data(), d_fp, fp.size(), s);
        return fp;
    };
    std::vector<int64_t> tstart;  // tile ranges over `order`
    if (rstart.size() > 20) {
        const std::vector<int64_t> fp = footprints(rstart, rlen);
        std::vector<int64_t> srt = fp;
        const size_t q = (size_t)(0.95 * (double)(srt.size() - 1));
        std::nth_element(srt.begin(), srt.begin() + q, srt.end());
        int64_t budget = srt[q];
        if (const char* e = std::getenv("CF_SMEM_BUDGET")) budget = std::min<int64_t>(budget, std::atoll(e));
        // final pieces: (start, len); pending over-budget pieces are split level by level
        std::vector<std::pair<int64_t, int32_t>> fin;
        std::vector<int64_t> ps;
        std::vector<int32_t> pl;
        for (size_t t = 0; t < rstart.size(); ++t) {
            if (fp[t] <= budget || rlen[t] <= 16) fin.push_back({rstart[t], rlen[t]});
            else {
                ps.push_back(rstart[t]);
                pl.push_back(rlen[t]);
            }
        }
        while (!ps.empty()) {
            std::vector<int64_t> hs;
            std::vector<int32_t> hl;
            for (size_t i = 0; i < ps.size(); ++i) {
                const int32_t h = pl[i] / 2;
                hs.push_back(ps[i]);
                hl.push_back(h);
                hs.push_back(ps[i] + h);
                hl.push_back(pl[i] - h);
            }
            const std::vector<int64_t> hf = footprints(hs, hl);
            ps.clear();
            pl.clear();
            for (size_t i = 0; i < hs.size(); ++i) {
                if (hl[i] <= 16 || hf[i] <= budget) fin.push_back({hs[i], hl[i]});
                else {
                    ps.push_back(hs[i]);
                    pl.push_back(hl[i]);
                }
            }
        }
        std::sort(fin.begin(), fin.end());
        for (auto& x : fin) tstart.push_back(x.first);
    } else {
        tstart = rstart;
    }
    tstart.push_back(Er);
    const int64_t nT = (int64_t)tstart.size() - 1;
    for (int64_t t = 0; t < nT; ++t)
        if (tstart[t + 1] - tstart[t] > kMaxTileElems)
            raise(CF_INVALID_ARG, "a tile holds more than 2048 elements (" + std::to_string(tstart[t + 1] - tstart[t]) + ")");
    int64_t* d_tstart = T.alloc<int64_t>(nT + 1);
    h2d(d_tstart, tstart.data(), nT + 1, s);
    seg_sort_keys(order, Er, d_tstart, nT, s);  // ascending id within a tile (BlockPlan)

    // ---- local node numbering: RCM label / given / first touch in tile order
    int32_t* local_of = T.alloc<int32_t>(N);
    int32_t* lnodes_full = T.alloc<int32_t>(N);
    uint8_t* mark = nullptr;
    if (W > 1) {
        mark = T.alloc<uint8_t>(N);
        DP_CHECK(cudaMemsetAsync(mark, 0, N, s));
        if (Er) k_mark<<<grid_of(4 * Er), 256, 0, s>>>(Er, order, m.tets, mark);
    }
    int64_t n_local = 0;
    if (o.node_order == CF_NODE_ORDER_TILE) {
        DBuf TT;
        unsigned long long* ft = TT.alloc<unsigned long long>(N);
        unsigned long long* ft2 = TT.alloc<unsigned long long>(N);
        int32_t* iv = TT.alloc<int32_t>(N);
        k_fill<<<grid_of(N), 256, 0, s>>>(N, ft, ~0ull);
        if (Er) k_first_touch<<<grid_of(4 * Er), 256, 0, s>>>(Er, order, m.tets, ft);
        k_iota<<<grid_of(N), 256, 0, s>>>(N, iv);
        sort_pairs(ft, ft2, iv, lnodes_full, N, 64, s);
        // nodes never touched sort last (key ~0)
        unsigned long long* cntp = TT.alloc<unsigned long long>(1);
        DP_CHECK(cudaMemsetAsync(cntp, 0, 8, s));
        {
            size_t tb = 0;
            DP_CHECK(cub::DeviceReduce::Sum(nullptr, tb, cub::TransformInputIterator<int64_t, NotMax, unsigned long long*>(ft2, NotMax{}), cntp, N, s));
            DBuf T3;
            void* tmp = T3.alloc<uint8_t>(tb);
            DP_CHECK(cub::DeviceReduce::Sum(tmp, tb, cub::TransformInputIterator<int64_t, NotMax, unsigned long long*>(ft2, NotMax{}), cntp, N, s));
            n_local = (int64_t)read1(cntp, s);
        }
        k_fill<<<grid_of(N), 256, 0, s>>>(N, local_of, -1);
        if (n_local) k_number_list<<<grid_of(n_local), 256, 0, s>>>(n_local, lnodes_full, local_of);
    } else {
        DBuf TT;
        int32_t* inv = TT.alloc<int32_t>(N);
        int32_t* flag = TT.alloc<int32_t>(N);
        int32_t* pos = TT.alloc<int32_t>(N + 1);
        const int32_t* lab = o.node_order == CF_NODE_ORDER_RCM ? d_label : nullptr;
        k_inv<<<grid_of(N), 256, 0, s>>>(N, lab, inv);
        k_flag_by_label<<<grid_of(N), 256, 0, s>>>(N, inv, mark, flag);
        excl_sum(flag, pos, N, s);
        n_local = read1(pos + N, s);
        k_number_by_label<<<grid_of(N), 256, 0, s>>>(N, inv, flag, pos, lnodes_full, local_of);
    }
    DP_CHECK(cudaGetLastError());
    if (n_local >= (1 << 28)) raise(CF_INVALID_ARG, "more than 2^28 nodes on one rank");
    rp.n_local = (int32_t)n_local;

    // ---- ghosts (sister nodes of this rank's interface facets that are not local) and the
    // multi-rank classification inputs: interface-facet records gathered to the host
    std::vector<int32_t> ifac;  // interface facets, ascending
    for (int32_t f = 0; f < F; ++f)
        if (S.facet_kind[f] >= 0 && S.P.kind[S.facet_kind[f]].interface) ifac.push_back(f);
    std::vector<int32_t> sis_nodes(4 * ifac.size()), sis_local(4 * ifac.size()), sis_part(ifac.size(), 0);
    std::vector<unsigned long long> sis_mask(4 * ifac.size(), 0);
    std::vector<int32_t> ghosts;
    if (W > 1 && !ifac.empty()) {
        DBuf TT;
        std::vector<int32_t> se(ifac.size());
        for (size_t i = 0; i < ifac.size(); ++i) se[i] = sister[ifac[i]];
        int32_t* d_se = TT.alloc<int32_t>(se.size());
        int32_t* d_sp = TT.alloc<int32_t>(se.size());
        h2d(d_se, se.data(), se.size(), s);
        k_gather_i32<<<grid_of((int64_t)se.size()), 256, 0, s>>>((int64_t)se.size(), d_se, d_part, d_sp);
        d2h(sis_part.data(), d_sp, se.size(), s);
        const int64_t n4 = 4 * (int64_t)se.size();  // the sister elements' corners (element ids may exceed 2^29)
        int32_t* d_sn = TT.alloc<int32_t>(n4);
        int32_t* d_sl = TT.alloc<int32_t>(n4);
        unsigned long long* d_sm = TT.alloc<unsigned long long>(n4);
        k_gather_corners<<<grid_of(n4), 256, 0, s>>>((int64_t)se.size(), d_se, m.tets, d_sn);
        k_gather_i32<<<grid_of(n4), 256, 0, s>>>(n4, d_sn, local_of, d_sl);
        k_gather_u64<<<grid_of(n4), 256, 0, s>>>(n4, d_sn, nmask, d_sm);
        d2h(sis_nodes.data(), d_sn, n4, s);
        d2h(sis_local.data(), d_sl, n4, s);
        d2h(sis_mask.data(), d_sm, n4, s);
        for (size_t i = 0; i < ifac.size(); ++i) {
            if (!in_rank_owner(ifac[i])) continue;
            for (int a = 0; a < 4; ++a)
                if (sis_local[4 * i + a] < 0) ghosts.push_back(sis_nodes[4 * i + a]);
        }
        std::sort(ghosts.begin(), ghosts.end());
        ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
        if (!ghosts.empty()) {
            std::vector<int32_t> gl(ghosts.size());
            for (size_t g = 0; g < ghosts.size(); ++g) gl[g] = (int32_t)(n_local + (int64_t)g);
            int32_t* d_g = TT.alloc<int32_t>(ghosts.size());
            int32_t* d_gl = TT.alloc<int32_t>(ghosts.size());
            h2d(d_g, ghosts.data(), ghosts.size(), s);
            h2d(d_gl, gl.data(), gl.size(), s);
            k_scatter_i32<<<grid_of((int64_t)ghosts.size()), 256, 0, s>>>((int64_t)ghosts.size(), d_g, d_gl, local_of);
            DP_CHECK(cudaStreamSynchronize(s));
        }
    }
    rp.n_ghost = (int32_t)ghosts.size();
    out.local_global = M.alloc<int32_t>(n_local + ghosts.size());
    DP_CHECK(cudaMemcpyAsync(out.local_global, lnodes_full, n_local * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    h2d(out.local_global + n_local, ghosts.data(), ghosts.size(), s);
    T.free(lnodes_full);
    const int32_t* lnodes = out.local_global;
    out.node_region = M.alloc<uint8_t>(n_local);
    int32_t* any_dir = T.alloc<int32_t>(1);
    DP_CHECK(cudaMemsetAsync(any_dir, 0, 4, s));
    if (n_local) k_lnode_attr<<<grid_of(n_local), 256, 0, s>>>(n_local, lnodes, m.node_region, DS.dir_of_node,
                                                               out.node_region, nullptr, any_dir);
    if (read1(any_dir, s)) {
        out.node_dir = M.alloc<int8_t>(n_local);
        k_lnode_attr<<<grid_of(n_local), 256, 0, s>>>(n_local, lnodes, m.node_region, DS.dir_of_node, out.node_region,
                                                      out.node_dir, any_dir);
    }
    c.local_of = local_of;
    c.lnode_region = out.node_region;
    c.lnode_dir = out.node_dir;

    // ---- pass 1: per-tile metadata, then the ordered tile nodes
    TileMeta* d_meta = T.alloc<TileMeta>(nT);
    int32_t* tn_off = T.alloc<int32_t>(nT + 1);
    int32_t* tnodes = nullptr;
    {
        int64_t mx = 1;
        for (int64_t t = 0; t < nT; ++t) mx = std::max<int64_t>(mx, tstart[t + 1] - tstart[t]);
        const int64_t wsi = 4 * mx + 16 * mx + 64;
        const int64_t batch = ws_batch(wsi, std::max<int64_t>(1, nT));
        DBuf TT;
        int32_t* ws = TT.alloc<int32_t>(batch * wsi);
        for (int64_t b0 = 0; b0 < nT; b0 += batch) {
            const int64_t b1 = std::min(nT, b0 + batch);
            k_pass1<<<(int)((b1 - b0 + 127) / 128), 128, 0, s>>>(c, order, d_tstart, b0, b1, ws, wsi, d_meta, nullptr, nullptr);
        }
        DP_CHECK(cudaGetLastError());
        int32_t* ns_arr = TT.alloc<int32_t>(nT);
        {
            std::vector<TileMeta> hm(nT);
            d2h(hm.data(), d_meta, nT, s);
            rp.tile_meta = hm;
            std::vector<int32_t> nsv(nT);
            int64_t sum_ns = 0;
            for (int64_t t = 0; t < nT; ++t) sum_ns += nsv[t] = hm[t].ns;
            if (sum_ns > INT32_MAX) raise(CF_INVALID_ARG, "more than 2^31 tile slots on one rank");
            h2d(ns_arr, nsv.data(), nT, s);
        }
        excl_sum(ns_arr, tn_off, nT, s);
        const int64_t tot = read1(tn_off + nT, s);
        tnodes = T.alloc<int32_t>(tot);
        for (int64_t b0 = 0; b0 < nT; b0 += batch) {
            const int64_t b1 = std::min(nT, b0 + batch);
            k_pass1<<<(int)((b1 - b0 + 127) / 128), 128, 0, s>>>(c, order, d_tstart, b0, b1, ws, wsi, d_meta, tn_off, tnodes);
        }
        DP_CHECK(cudaGetLastError());
        DP_CHECK(cudaStreamSynchronize(s));
    }
    rp.n_tiles = (int32_t)nT;
    // tiles touching each node (tile-private test), rank-shared nodes, border tiles
    int32_t* ntiles_of = T.alloc<int32_t>(std::max<int64_t>(1, n_local));
    DP_CHECK(cudaMemsetAsync(ntiles_of, 0, std::max<int64_t>(1, n_local) * sizeof(int32_t), s));
    if (nT) k_ntiles<<<grid_of(nT), 256, 0, s>>>(nT, tn_off, tnodes, ntiles_of);
    uint8_t* shared_node = nullptr;
    rp.tile_border.assign(nT, 0);
    if (W > 1) {
        shared_node = T.alloc<uint8_t>(std::max<int64_t>(1, n_local));
        if (n_local) k_shared_node<<<grid_of(n_local), 256, 0, s>>>(n_local, lnodes, nmask, shared_node);
        uint8_t* bd = T.alloc<uint8_t>(std::max<int64_t>(1, nT));
        if (nT) k_border<<<grid_of(nT), 256, 0, s>>>(nT, tn_off, tnodes, shared_node, bd);
        d2h(rp.tile_border.data(), bd, nT, s);
    }
    c.ntiles_of = ntiles_of;
    c.shared_node = shared_node;

    // ---- offsets (host, O(tiles))
    for (int64_t t = 0; t < nT; ++t) {
        const TileMeta& tm = rp.tile_meta[t];
        const TileLayout L(tm, S.temp_dep, coords);
        if (4 * tm.ne + 4 * tm.nf > 65535 || tm.ncsr > 65535 || tm.ne > 1024 || L.max_operand() > 0x7fff)
            raise(CF_INVALID_ARG, "tile too large for 16-bit slot / operand indices (at most 1024 tets per tile)");
    }
    rp.tile_slot_off.assign(nT + 1, 0);
    rp.blob_off.assign(nT + 1, 0);
    rp.elem_off.assign(tstart.begin(), tstart.end());
    TileCaps caps{1, 1, 0, 0};
    for (int64_t t = 0; t < nT; ++t) {
        const TileMeta& tm = rp.tile_meta[t];
        const TileLayout L(tm, S.temp_dep, coords);
        rp.blob_off[t + 1] = rp.blob_off[t] + L.total;
        rp.tile_slot_off[t + 1] = rp.tile_slot_off[t] + (int32_t)cf_round(tm.ns, 2);
        rp.max_elems = std::max(rp.max_elems, tm.ne);
        rp.max_slots = std::max(rp.max_slots, (int32_t)cf_round(tm.ns, 2));
        rp.max_facets = std::max(rp.max_facets, tm.nf);
        rp.max_blob = std::max<int64_t>(rp.max_blob, L.bytes);
        rp.max_scratch = std::max<int64_t>(rp.max_scratch, L.scratch);
        caps.ne = std::max(caps.ne, tm.ne);
        caps.ns = std::max(caps.ns, tm.ns);
        caps.nf = std::max(caps.nf, tm.nf);
        caps.ncsr = std::max(caps.ncsr, tm.ncsr);
    }
    rp.blob_bytes = rp.blob_off[nT];
    const int64_t S_tot = rp.tile_slot_off[nT];
    out.S_tot = S_tot;
    out.E_r = Er;
    int64_t* d_boff = T.alloc<int64_t>(nT + 1);
    int32_t* d_soff = M.alloc<int32_t>(nT + 1);
    h2d(d_boff, rp.blob_off.data(), nT + 1, s);
    h2d(d_soff, rp.tile_slot_off.data(), nT + 1, s);

    // ---- packing: every non-geometry section, one tile per thread; then the geometry
    out.blob = M.alloc<uint8_t>((size_t)std::max<int64_t>(16, rp.blob_bytes));
    DP_CHECK(cudaMemsetAsync(out.blob, 0, (size_t)std::max<int64_t>(16, rp.blob_bytes), s));
    out.slot_node = M.alloc<int32_t>(S_tot);
    out.elem_global = M.alloc<int32_t>(Er);
    unsigned long long* counts = T.alloc<unsigned long long>(2);
    DP_CHECK(cudaMemsetAsync(counts, 0, 16, s));
    {
        PackK a;
        a.c = c;
        a.order = order;
        a.tstart = d_tstart;
        a.meta = d_meta;
        a.tn_off = tn_off;
        a.tnodes = tnodes;
        a.blob_off = d_boff;
        a.slot_off = d_soff;
        a.blob = out.blob;
        a.slot_node = out.slot_node;
        a.elem_global = out.elem_global;
        a.ws_ints = tile_ws_ints(caps);
        a.counts = counts;
        const int64_t batch = ws_batch(a.ws_ints, std::max<int64_t>(1, nT));
        DBuf TT;
        a.ws = TT.alloc<int32_t>(batch * a.ws_ints);
        for (int64_t b0 = 0; b0 < nT; b0 += batch) {
            const int64_t b1 = std::min(nT, b0 + batch);
            k_pack<<<(int)((b1 - b0 + 127) / 128), 128, 0, s>>>(a, b0, b1);
        }
        DP_CHECK(cudaGetLastError());
        DP_CHECK(cudaStreamSynchronize(s));
    }
    {
        unsigned long long h[2];
        d2h(h, counts, 2, s);
        rp.n_if_facets = (int64_t)h[0];
        rp.n_bc_facets = (int64_t)h[1];
    }
    if (nT)
        k_fill_geom<<<(int)nT, 128, 0, s>>>(d_meta, d_boff, d_tstart, out.elem_global, m.tets, m.coords, d_soff,
                                           out.slot_node, out.local_global, out.blob, S.temp_dep, coords);
    DP_CHECK(cudaGetLastError());
    T.free(order);
    T.free(tnodes);

    // ---- merge lists: ascending tile (slot index) per node (merge_offsets/merge_entries
    // blocked.hpp:294-307); shared list ordered by first partial
    out.merge_off = M.alloc<int32_t>(n_local + 1);
    out.merge_idx = M.alloc<int32_t>(S_tot);
    {
        DBuf TT;
        int32_t* k0 = TT.alloc<int32_t>(S_tot);
        int32_t* k1 = TT.alloc<int32_t>(S_tot);
        int32_t* v0 = TT.alloc<int32_t>(S_tot);
        int32_t* cnt = TT.alloc<int32_t>(std::max<int64_t>(1, n_local));
        DP_CHECK(cudaMemsetAsync(cnt, 0, std::max<int64_t>(1, n_local) * sizeof(int32_t), s));
        if (S_tot) k_merge_keys<<<grid_of(S_tot), 256, 0, s>>>(S_tot, out.slot_node, (int32_t)n_local, k0, v0, cnt);
        sort_pairs(k0, k1, v0, out.merge_idx, S_tot, 29, s);
        excl_sum(cnt, out.merge_off, n_local, s);
        const int64_t used = read1(out.merge_off + n_local, s);
        if (used < S_tot) k_zero_tail<<<grid_of(S_tot - used), 256, 0, s>>>(used, S_tot, out.merge_idx);
    }
    {
        DBuf TT;
        uint64_t* k0 = TT.alloc<uint64_t>(std::max<int64_t>(1, n_local));
        uint64_t* k1 = TT.alloc<uint64_t>(std::max<int64_t>(1, n_local));
        int32_t* v0 = TT.alloc<int32_t>(std::max<int64_t>(1, n_local));
        int32_t* v1 = TT.alloc<int32_t>(std::max<int64_t>(1, n_local));
        unsigned long long* nsh = TT.alloc<unsigned long long>(1);
        DP_CHECK(cudaMemsetAsync(nsh, 0, 8, s));
        if (n_local)
            k_shared_keys<<<grid_of(n_local), 256, 0, s>>>(n_local, ntiles_of, shared_node, out.merge_off, out.merge_idx, k0,
                                                           v0, nsh);
        sort_pairs(k0, k1, v0, v1, n_local, 64, s);
        const int64_t n_sh = (int64_t)read1(nsh, s);
        out.n_shared_list = n_sh;
        rp.n_private = n_local - n_sh;
        out.shared_list = M.alloc<int32_t>(std::max<int64_t>(1, n_sh));
        DP_CHECK(cudaMemcpyAsync(out.shared_list, v1, n_sh * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        out.shared_rec = M.alloc<int4>(2 * std::max<int64_t>(1, n_sh));
        out.shared_rec2 = M.alloc<int2>(std::max<int64_t>(1, n_sh));
        DP_CHECK(cudaMemsetAsync(out.shared_rec, 0, 2 * std::max<int64_t>(1, n_sh) * sizeof(int4), s));
        DP_CHECK(cudaMemsetAsync(out.shared_rec2, 0, std::max<int64_t>(1, n_sh) * sizeof(int2), s));
        unsigned long long* parts = TT.alloc<unsigned long long>(1);
        DP_CHECK(cudaMemsetAsync(parts, 0, 8, s));
        if (n_sh) k_shared_rec<<<grid_of(n_sh), 256, 0, s>>>(n_sh, out.shared_list, out.merge_off, out.merge_idx,
                                                            out.shared_rec, out.shared_rec2, parts);
        out.merge_parts = (int64_t)read1(parts, s);
    }

    // ---- multi-rank exchange (classify_nodes partition.hpp:305-367; external_from :346-354):
    // O(interface) lists on the host, the build_rank_plan logic
    if (W > 1) {
        std::vector<int32_t> sh_g, sh_l;
        std::vector<unsigned long long> sh_m;
        {
            DBuf TT;
            const int64_t cap = std::max<int64_t>(1, n_local);
            int32_t* g = TT.alloc<int32_t>(cap);
            int32_t* l = TT.alloc<int32_t>(cap);
            unsigned long long* mm = TT.alloc<unsigned long long>(cap);
            unsigned long long* cnt = TT.alloc<unsigned long long>(1);
            DP_CHECK(cudaMemsetAsync(cnt, 0, 8, s));
            if (n_local) k_select_shared<<<grid_of(n_local), 256, 0, s>>>(n_local, lnodes, shared_node, g, l, mm, nmask, cnt);
            const int64_t k = (int64_t)read1(cnt, s);
            sh_g.resize(k);
            sh_l.resize(k);
            sh_m.resize(k);
            d2h(sh_g.data(), g, k, s);
            d2h(sh_l.data(), l, k, s);
            d2h(sh_m.data(), mm, k, s);
        }
        std::vector<int64_t> ordv(sh_g.size());
        std::iota(ordv.begin(), ordv.end(), 0);
        std::sort(ordv.begin(), ordv.end(), [&](int64_t a, int64_t b) { return sh_g[a] < sh_g[b]; });
        rp.n_shared = (int64_t)sh_g.size();
        std::vector<int32_t> node_shared_idx(sh_g.size());  // shared index -> local
        std::map<int32_t, RankPlan::Neighbor> nb;
        for (size_t i = 0; i < ordv.size(); ++i) {
            const int64_t j = ordv[i];
            node_shared_idx[i] = sh_l[j];
            unsigned long long b = sh_m[j];
            while (b) {
                const int32_t q = __builtin_ctzll(b);
                b &= b - 1;
                if (q != rank) nb[q].shared.push_back(sh_l[j]);
            }
        }
        auto node_on = [&](size_t fi, int a, int32_t p) { return (sis_mask[4 * fi + a] >> p) & 1ull; };
        auto ext_need = [&](int32_t p, int32_t q, bool locals) {
            std::vector<std::pair<int32_t, int32_t>> v;  // (global, local)
            for (size_t i = 0; i < ifac.size(); ++i) {
                if (owner_part[ifac[i]] != p || sis_part[i] != q) continue;
                for (int a = 0; a < 4; ++a)
                    if (!node_on(i, a, p)) v.push_back({sis_nodes[4 * i + a], locals ? sis_local[4 * i + a] : -1});
            }
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            return v;
        };
        // ghost local ids: n_local + index in the sorted ghost list
        auto ghost_local = [&](int32_t n) {
            return (int32_t)(n_local + (std::lower_bound(ghosts.begin(), ghosts.end(), n) - ghosts.begin()));
        };
        for (int32_t q = 0; q < W; ++q) {
            if (q == rank) continue;
            const auto from = ext_need(rank, q, false);
            const auto to = ext_need(q, rank, true);
            if (from.empty() && to.empty() && !nb.count(q)) continue;
            auto& x = nb[q];
            for (const auto& n : from) x.ext_from.push_back(ghost_local(n.first));
            for (const auto& n : to) {
                if (n.second < 0 || n.second >= n_local) raise(CF_PROTOCOL, "external node not local to sender");
                x.ext_to.push_back(n.second);
            }
        }
        rp.send_off.push_back(0);
        rp.recv_off.push_back(0);
        for (auto& kv : nb) {
            kv.second.rank = kv.first;
            rp.nbrs.push_back(kv.second);
            const auto& x = rp.nbrs.back();
            rp.send_off.push_back(rp.send_off.back() + 2 * (int64_t)x.shared.size() + (int64_t)x.ext_to.size());
            rp.recv_off.push_back(rp.recv_off.back() + 2 * (int64_t)x.shared.size() + (int64_t)x.ext_from.size());
        }
        rp.send_len = rp.send_off.back();
        rp.recv_len = rp.recv_off.back();
        // combine lists per shared node: ascending rank, own included (build_rank_plan: every
        // replica sums in the same order, so the shared-node copies stay bitwise identical)
        std::map<int32_t, int32_t> shared_of_local;
        for (size_t i = 0; i < node_shared_idx.size(); ++i) shared_of_local[node_shared_idx[i]] = (int32_t)i;
        std::vector<std::vector<std::array<int32_t, 3>>> src(node_shared_idx.size());
        for (size_t i = 0; i < src.size(); ++i) src[i].push_back({rank, -1, -1});
        for (size_t k = 0; k < rp.nbrs.size(); ++k) {
            const auto& x = rp.nbrs[k];
            const int32_t ns = (int32_t)x.shared.size();
            for (int32_t j = 0; j < ns; ++j)
                src[shared_of_local[x.shared[j]]].push_back(
                    {x.rank, (int32_t)(rp.recv_off[k] + j), (int32_t)(rp.recv_off[k] + ns + j)});
        }
        rp.shared_off.assign(src.size() + 1, 0);
        for (size_t i = 0; i < src.size(); ++i) {
            std::sort(src[i].begin(), src[i].end());
            rp.shared_off[i + 1] = rp.shared_off[i] + (int32_t)src[i].size();
            for (auto& pr : src[i]) {
                rp.shared_src.push_back(pr[1]);
                rp.shared_src_r.push_back(pr[2]);
            }
        }
        rp.ghost_src.assign(rp.n_ghost, -1);
        for (size_t k = 0; k < rp.nbrs.size(); ++k) {
            const auto& x = rp.nbrs[k];
            const int64_t base = rp.recv_off[k] + 2 * (int64_t)x.shared.size();
            for (size_t j = 0; j < x.ext_from.size(); ++j) {
                const int32_t g = x.ext_from[j] - (int32_t)n_local;
                if (g >= 0 && rp.ghost_src[g] < 0) rp.ghost_src[g] = (int32_t)(base + (int64_t)j);
            }
        }
        for (int32_t g = 0; g < rp.n_ghost; ++g)
            if (rp.ghost_src[g] < 0) raise(CF_PROTOCOL, "ghost node without a provider");
        // device tables
        std::vector<int32_t> ns_full(n_local, -1);
        for (size_t i = 0; i < node_shared_idx.size(); ++i) ns_full[node_shared_idx[i]] = (int32_t)i;
        rp.node_shared = ns_full;
        out.node_shared = M.alloc<int32_t>(std::max<int64_t>(1, n_local));
        h2d(out.node_shared, ns_full.data(), n_local, s);
        out.shared_off = M.alloc<int32_t>(rp.shared_off.size());
        h2d(out.shared_off, rp.shared_off.data(), rp.shared_off.size(), s);
        out.shared_src = M.alloc<int32_t>(rp.shared_src.size());
        h2d(out.shared_src, rp.shared_src.data(), rp.shared_src.size(), s);
        out.shared_src_r = M.alloc<int32_t>(rp.shared_src_r.size());
        h2d(out.shared_src_r, rp.shared_src_r.data(), rp.shared_src_r.size(), s);
        out.ghost_src = M.alloc<int32_t>(rp.ghost_src.size());
        h2d(out.ghost_src, rp.ghost_src.data(), rp.ghost_src.size(), s);
    }
    DP_CHECK(cudaStreamSynchronize(s));
}

// the device plan's arrays downloaded into a host RankPlan (test instrumentation: digests)
void download_dev_rank_plan(const DevRankPlan& p, bool tdep, bool coords, cudaStream_t s, RankPlan& rp) {
    rp = p.H;
    const int64_t nT = rp.n_tiles;
    std::vector<uint8_t> blob((size_t)rp.blob_bytes);
    d2h(blob.data(), p.blob, blob.size(), s);
    rp.rest_off.assign(nT + 1, 0);
    for (int64_t t = 0; t < nT; ++t)
        rp.rest_off[t + 1] = rp.rest_off[t] + TileLayout(rp.tile_meta[t], tdep, coords).staged_bytes();
    rp.blob.resize(rp.rest_off[nT]);
    for (int64_t t = 0; t < nT; ++t) {
        const TileLayout L(rp.tile_meta[t], tdep, coords);
        std::memcpy(rp.blob.data() + rp.rest_off[t], blob.data() + rp.blob_off[t] + L.stage, L.staged_bytes());
    }
    rp.elem_global.resize(p.E_r);
    d2h(rp.elem_global.data(), p.elem_global, p.E_r, s);
    rp.slot_node.resize(p.S_tot);
    d2h(rp.slot_node.data(), p.slot_node, p.S_tot, s);
    rp.local_global.resize((size_t)rp.n_local + rp.n_ghost);
    d2h(rp.local_global.data(), p.local_global, rp.local_global.size(), s);
    rp.node_region.resize(rp.n_local);
    d2h(rp.node_region.data(), p.node_region, rp.n_local, s);
    rp.node_dir.clear();
    if (p.node_dir) {
        rp.node_dir.resize(rp.n_local);
        d2h(rp.node_dir.data(), p.node_dir, rp.n_local, s);
    }
    rp.merge_off.resize((size_t)rp.n_local + 1);
    d2h(rp.merge_off.data(), p.merge_off, rp.merge_off.size(), s);
    rp.merge_idx.resize(p.S_tot);
    d2h(rp.merge_idx.data(), p.merge_idx, p.S_tot, s);
    rp.shared_list.resize(p.n_shared_list);
    d2h(rp.shared_list.data(), p.shared_list, p.n_shared_list, s);
}

}  // namespace cfb
