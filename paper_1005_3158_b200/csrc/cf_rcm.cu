// cf_rcm.cu — the RCM reordering pass on the B200 (rcm_permutation reorder.hpp:127-148, over
// build_node_graph :17-24), reproducing the reference permutation exactly.
//
// The reference is a sequential Cuthill-McKee BFS: each visited vertex appends its not yet seen
// neighbours sorted by (degree, id) (bfs_levels :54-88); components are taken by ascending
// smallest id, each rooted at a George-Liu pseudo-peripheral vertex (:91-120); the order is
// reversed at the end. The order within BFS level L+1 is therefore fixed by the level-L
// position of each vertex's FIRST discoverer, then (degree, id) -- which a level-synchronous
// BFS computes in parallel:
//   claim   every level-L vertex at position p atomically min-claims its unseen neighbours: the
//           winner is the first discoverer;
//   count   each level-L vertex counts the neighbours it won;
//   scan    exclusive prefix sum of the counts (the level's output offsets);
//   emit    each level-L vertex writes its won neighbours, sorted by (degree, id), at its offset
//           and marks them seen.
// No global sort is needed: a vertex's won set is at most its degree.
//
// The node graph is built on the device as a CSR of unique neighbours (node -> incident
// elements -> the other three nodes, deduplicated per node), so the graph never exists on the
// host: cfg5 (135.6 M nodes, ~1.9 G directed edges) needs ~35 GB of device memory for the
// pass, freed before the plan is uploaded, against ~80 GB of host memory for the host graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "cf_internal.hpp"

namespace cfb {
namespace {

#define RCM_CHECK(x)                                                                                  \
    do {                                                                                              \
        cudaError_t e_ = (x);                                                                         \
        if (e_ != cudaSuccess) raise(CF_CUDA, std::string("rcm: ") + #x + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr int kLocal = 64;  // unique-neighbour list held per thread before the slow path

// ---- node -> element incidence
__global__ void incidence_count(int64_t E, const int32_t* __restrict__ tets, int32_t* cnt) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 4 * E; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[tets[k]], 1);
}
__global__ void incidence_fill(int64_t E, const int32_t* __restrict__ tets, int64_t* cursor, int32_t* n2e) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < 4 * E; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pos = (int64_t)atomicAdd((unsigned long long*)&cursor[tets[k]], 1ull);
        n2e[pos] = (int32_t)(k >> 2);
    }
}

// unique neighbours of v (the other nodes of its elements): visit(w) once per w.
// Fast path: a per-thread list of up to kLocal; beyond it, "first occurrence" scans.
template <class F>
__device__ __forceinline__ int for_each_neighbor(int32_t v, const int64_t* __restrict__ ioff,
                                                 const int32_t* __restrict__ n2e, const int32_t* __restrict__ tets,
                                                 F visit) {
    int32_t u[kLocal];
    int nu = 0;
    bool spill = false;
    const int64_t b = ioff[v], e = ioff[v + 1];
    for (int64_t j = b; j < e && !spill; ++j) {
        const int4 t = __ldg((const int4*)tets + n2e[j]);
        const int32_t q[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int32_t w = q[a];
            if (w == v) continue;
            bool dup = false;
            for (int i = 0; i < nu; ++i) dup |= u[i] == w;
            if (dup) continue;
            if (nu == kLocal) {
                spill = true;
                break;
            }
            u[nu++] = w;
        }
    }
    if (!spill) {
        for (int i = 0; i < nu; ++i) visit(u[i]);
        return nu;
    }
    // high-degree vertex: w counts at its first occurrence in the incidence scan
    int n = 0;
    for (int64_t j = b; j < e; ++j) {
        const int4 t = __ldg((const int4*)tets + n2e[j]);
        const int32_t q[4] = {t.x, t.y, t.z, t.w};
        for (int a = 0; a < 4; ++a) {
            const int32_t w = q[a];
            if (w == v) continue;
            bool seen_before = false;
            for (int64_t j2 = b; j2 <= j && !seen_before; ++j2) {
                const int4 t2 = __ldg((const int4*)tets + n2e[j2]);
                const int32_t q2[4] = {t2.x, t2.y, t2.z, t2.w};
                const int lim = j2 == j ? a : 4;
                for (int a2 = 0; a2 < lim; ++a2) seen_before |= q2[a2] == w;
            }
            if (!seen_before) {
                visit(w);
                ++n;
            }
        }
    }
    return n;
}

__global__ void graph_degree(int32_t N, const int64_t* ioff, const int32_t* n2e, const int32_t* tets, int32_t* deg) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x)
        deg[v] = for_each_neighbor(v, ioff, n2e, tets, [](int32_t) {});
}
__global__ void graph_fill(int32_t N, const int64_t* ioff, const int32_t* n2e, const int32_t* tets,
                           const int64_t* goff, int32_t* adj) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
        int32_t* out = adj + goff[v];
        int k = 0;
        for_each_neighbor(v, ioff, n2e, tets, [&](int32_t w) { out[k++] = w; });
    }
}

// ---- exclusive prefix sum of int32 counts into int64 offsets (out[n] = total), multi-block:
// per-block sums, a scan of the block sums (recursively), then the block-local scans
constexpr int kScanThreads = 1024, kScanItems = 4, kScanTile = kScanThreads * kScanItems;

template <class In>
__device__ int64_t block_exclusive_scan(int64_t v, int64_t* sh) {
    // Hillis-Steele over the block's per-thread sums
    const int t = threadIdx.x;
    sh[t] = v;
    __syncthreads();
    for (int o = 1; o < kScanThreads; o <<= 1) {
        const int64_t x = t >= o ? sh[t - o] : 0;
        __syncthreads();
        sh[t] += x;
        __syncthreads();
    }
    const int64_t incl = sh[t];
    __syncthreads();
    return incl - v;
}

template <class In>
__global__ void __launch_bounds__(kScanThreads) scan_tiles(int64_t n, const In* __restrict__ in, int64_t* out,
                                                          int64_t* block_sums) {
    __shared__ int64_t sh[kScanThreads];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int64_t x[kScanItems], s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        x[i] = base + i < n ? (int64_t)in[base + i] : 0;
        s += x[i];
    }
    int64_t run = block_exclusive_scan<In>(s, sh);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = run;
        run += x[i];
    }
    if (threadIdx.x == kScanThreads - 1) block_sums[blockIdx.x] = run;
}
__global__ void scan_add(int64_t n, int64_t* out, const int64_t* block_off) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    const int64_t add = block_off[blockIdx.x];
    for (int i = threadIdx.x; i < kScanTile && base + i < n; i += blockDim.x) out[base + i] += add;
}

struct DevBuf {
    std::vector<void*> p;
    template <class T>
    T* alloc(size_t n) {
        void* q = nullptr;
        RCM_CHECK(cudaMalloc(&q, std::max<size_t>(1, n) * sizeof(T)));
        p.push_back(q);
        return (T*)q;
    }
    void free(void* q) {
        auto it = std::find(p.begin(), p.end(), q);
        if (it != p.end()) {
            cudaFree(q);
            p.erase(it);
        }
    }
    ~DevBuf() {
        for (void* q : p) cudaFree(q);
    }
};

// scan workspace for up to n_max elements: per recursion level the block sums and their offsets
// (allocated once per RCM pass: the BFS scans every level)
struct ScanWs {
    std::vector<int64_t*> sums, offs;
};
ScanWs make_scan_ws(DevBuf& B, int64_t n_max) {
    ScanWs w;
    for (int64_t n = n_max;;) {
        const int64_t blocks = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
        w.sums.push_back(B.alloc<int64_t>(blocks + 1));
        w.offs.push_back(B.alloc<int64_t>(blocks + 1));
        if (blocks == 1) break;
        n = blocks;
    }
    return w;
}

// out[0..n) = exclusive scan of in[0..n), out[n] = total (out has n + 1 entries); asynchronous
template <class In>
void exclusive_scan(const In* in, int64_t n, int64_t* out, cudaStream_t s, const ScanWs& w, size_t lvl = 0) {
    if (lvl >= w.sums.size()) raise(CF_INVALID_ARG, "rcm: scan workspace too small");
    const int64_t blocks = std::max<int64_t>(1, (n + kScanTile - 1) / kScanTile);
    int64_t* sums = w.sums[lvl];
    scan_tiles<In><<<(unsigned)blocks, kScanThreads, 0, s>>>(n, in, out, sums);
    RCM_CHECK(cudaGetLastError());
    if (blocks > 1) {
        int64_t* soff = w.offs[lvl];
        exclusive_scan<int64_t>(sums, blocks, soff, s, w, lvl + 1);
        scan_add<<<(unsigned)blocks, 256, 0, s>>>(n, out, soff);
        RCM_CHECK(cudaGetLastError());
        RCM_CHECK(cudaMemcpyAsync(out + n, soff + blocks, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    } else {
        RCM_CHECK(cudaMemcpyAsync(out + n, sums, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    }
}

// ---- BFS pieces
// pseudo-peripheral BFS level: unseen neighbours of the frontier join the next level (set only)
__global__ void pp_expand(int32_t nf, const int32_t* __restrict__ front, const int64_t* __restrict__ goff,
                          const int32_t* __restrict__ adj, int32_t* dist, int32_t d, int32_t* next, int32_t* nnext) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
        const int32_t v = front[i];
        for (int64_t j = goff[v]; j < goff[v + 1]; ++j) {
            const int32_t u = adj[j];
            if (dist[u] < 0 && atomicCAS(&dist[u], -1, d) == -1) next[atomicAdd(nnext, 1)] = u;
        }
    }
}
// argmin over a vertex set of (degree, id), as a 64-bit key
__global__ void min_deg_id(int32_t n, const int32_t* __restrict__ set, const int32_t* __restrict__ deg,
                           unsigned long long* best) {
    unsigned long long m = ~0ull;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int32_t v = set[i];
        const unsigned long long k = (unsigned long long)(uint32_t)deg[v] << 32 | (uint32_t)v;
        m = k < m ? k : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
        m = x < m ? x : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(best, m);
}
// Cuthill-McKee level: first-discoverer claims (the level-local position of the parent)
__global__ void cm_claim(int32_t nf, const int32_t* __restrict__ front, const int64_t* __restrict__ goff,
                         const int32_t* __restrict__ adj, const int32_t* __restrict__ seen, int32_t* claim) {
    for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nf; p += gridDim.x * blockDim.x) {
        const int32_t v = front[p];
        for (int64_t j = goff[v]; j < goff[v + 1]; ++j) {
            const int32_t u = adj[j];
            if (!seen[u]) atomicMin(&claim[u], p);
        }
    }
}
__global__ void cm_count(int32_t nf, const int32_t* __restrict__ front, const int64_t* __restrict__ goff,
                         const int32_t* __restrict__ adj, const int32_t* __restrict__ seen,
                         const int32_t* __restrict__ claim, int32_t* cnt) {
    for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nf; p += gridDim.x * blockDim.x) {
        const int32_t v = front[p];
        int32_t c = 0;
        for (int64_t j = goff[v]; j < goff[v + 1]; ++j) {
            const int32_t u = adj[j];
            c += !seen[u] && claim[u] == p;
        }
        cnt[p] = c;
    }
}
// the parent's won neighbours sorted by (degree, id) -- bfs_levels' `fresh` order -- written at
// its offset of the next level; they become seen (only their winner ever writes them)
__global__ void cm_emit(int32_t nf, const int32_t* __restrict__ front, const int64_t* __restrict__ goff,
                        const int32_t* __restrict__ adj, const int32_t* __restrict__ deg, int32_t* seen,
                        const int32_t* __restrict__ claim, const int64_t* __restrict__ off, int32_t* out) {
    for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nf; p += gridDim.x * blockDim.x) {
        const int32_t v = front[p];
        int32_t* dst = out + off[p];
        const int32_t n = (int32_t)(off[p + 1] - off[p]);
        int k = 0;
        for (int64_t j = goff[v]; j < goff[v + 1]; ++j) {
            const int32_t u = adj[j];
            if (seen[u] || claim[u] != p) continue;
            // insertion into dst[0..k) by (degree, id)
            const int32_t du = deg[u];
            int i = k++;
            while (i > 0) {
                const int32_t w = dst[i - 1];
                const int32_t dw = deg[w];
                if (dw < du || (dw == du && w < u)) break;
                dst[i] = w;
                --i;
            }
            dst[i] = u;
        }
        (void)n;
        for (int i = 0; i < k; ++i) seen[dst[i]] = 1;
    }
}
// smallest unseen vertex id in [lo, hi), or INT32_MAX
__global__ void first_unseen(int32_t lo, int32_t hi, const int32_t* __restrict__ seen, int32_t* res) {
    int32_t m = INT32_MAX;
    for (int32_t v = lo + blockIdx.x * blockDim.x + threadIdx.x; v < hi; v += gridDim.x * blockDim.x)
        if (!seen[v]) {
            m = v;
            break;  // strided: later v of this thread are larger
        }
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m != INT32_MAX) atomicMin(res, m);
}
__global__ void reverse_labels(int32_t n, const int32_t* __restrict__ order, int32_t* new_of_old) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        new_of_old[order[i]] = n - 1 - i;
}

unsigned grid_for(int64_t n, int threads = 256) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16));
}

}  // namespace

// the pass over device-resident tets; new_of_old: device array [N] (the labels)
void rcm_labels_device(int32_t N, int64_t E, const int32_t* tets, int32_t seed, cudaStream_t s, int32_t* new_of_old) {
    if (N == 0) return;
    DevBuf B;
    // ---- node graph (build_node_graph reorder.hpp:17-24) on the device
    int32_t* icnt = B.alloc<int32_t>(N);
    RCM_CHECK(cudaMemsetAsync(icnt, 0, (size_t)N * sizeof(int32_t), s));
    incidence_count<<<grid_for(4 * E), 256, 0, s>>>(E, tets, icnt);
    int64_t* ioff = B.alloc<int64_t>((size_t)N + 1);
    const ScanWs ws = make_scan_ws(B, N);
    exclusive_scan<int32_t>(icnt, N, ioff, s, ws);
    int64_t* cursor = B.alloc<int64_t>((size_t)N + 1);
    RCM_CHECK(cudaMemcpyAsync(cursor, ioff, ((size_t)N + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    int32_t* n2e = B.alloc<int32_t>(4 * (size_t)E);
    incidence_fill<<<grid_for(4 * E), 256, 0, s>>>(E, tets, cursor, n2e);
    B.free(cursor);
    int32_t* deg = icnt;  // reused: incidence counts are consumed by the scan
    graph_degree<<<grid_for(N, 128), 128, 0, s>>>(N, ioff, n2e, tets, deg);
    RCM_CHECK(cudaGetLastError());
    int64_t* goff = B.alloc<int64_t>((size_t)N + 1);
    exclusive_scan<int32_t>(deg, N, goff, s, ws);
    int64_t n_adj = 0;
    RCM_CHECK(cudaMemcpyAsync(&n_adj, goff + N, sizeof n_adj, cudaMemcpyDeviceToHost, s));
    RCM_CHECK(cudaStreamSynchronize(s));
    int32_t* adj = B.alloc<int32_t>((size_t)n_adj);
    graph_fill<<<grid_for(N, 128), 128, 0, s>>>(N, ioff, n2e, tets, goff, adj);
    RCM_CHECK(cudaGetLastError());
    RCM_CHECK(cudaStreamSynchronize(s));
    B.free(n2e);
    B.free(ioff);

    // ---- BFS state
    int32_t* seen = B.alloc<int32_t>(N);
    int32_t* dist = B.alloc<int32_t>(N);
    int32_t* claim = B.alloc<int32_t>(N);
    int32_t* order = B.alloc<int32_t>(N);  // Cuthill-McKee order, all components
    int32_t* fa = B.alloc<int32_t>(N);     // pseudo-peripheral frontiers
    int32_t* fb = B.alloc<int32_t>(N);
    int32_t* cnt = B.alloc<int32_t>(N);
    int64_t* loff = B.alloc<int64_t>((size_t)N + 1);
    int32_t* dscal = B.alloc<int32_t>(2);
    unsigned long long* dbest = B.alloc<unsigned long long>(1);
    RCM_CHECK(cudaMemsetAsync(seen, 0, (size_t)N * sizeof(int32_t), s));
    RCM_CHECK(cudaMemsetAsync(claim, 0x7f, (size_t)N * sizeof(int32_t), s));  // 0x7f7f7f7f > any position
    // BFS over the whole component of `start` (set semantics) into dist; returns (depth, last level in fa/fb)
    auto bfs_sets = [&](int32_t start, int32_t*& last, int32_t& nlast) -> int64_t {
        RCM_CHECK(cudaMemsetAsync(dist, 0xff, (size_t)N * sizeof(int32_t), s));
        const int32_t zero = 0;
        RCM_CHECK(cudaMemcpyAsync(dist + start, &zero, sizeof zero, cudaMemcpyHostToDevice, s));
        RCM_CHECK(cudaMemcpyAsync(fa, &start, sizeof start, cudaMemcpyHostToDevice, s));
        int32_t *f = fa, *g = fb;
        int32_t nf = 1;
        int64_t depth = 0;
        last = f;
        nlast = 1;
        for (;;) {
            RCM_CHECK(cudaMemsetAsync(dscal, 0, sizeof(int32_t), s));
            pp_expand<<<grid_for(nf), 256, 0, s>>>(nf, f, goff, adj, dist, (int32_t)(depth + 1), g, dscal);
            int32_t nn = 0;
            RCM_CHECK(cudaMemcpyAsync(&nn, dscal, sizeof nn, cudaMemcpyDeviceToHost, s));
            RCM_CHECK(cudaStreamSynchronize(s));
            if (nn == 0) break;
            ++depth;
            std::swap(f, g);
            nf = nn;
            last = f;
            nlast = nf;
        }
        return depth;
    };
    // pseudo_peripheral reorder.hpp:91-120
    auto pseudo_peripheral = [&](int32_t start) {
        int32_t node = start;
        int64_t ecc = -1;
        for (;;) {
            int32_t* last = nullptr;
            int32_t nlast = 0;
            const int64_t depth = bfs_sets(node, last, nlast);
            if (depth <= ecc) return node;
            ecc = depth;
            const unsigned long long init = ~0ull;
            RCM_CHECK(cudaMemcpyAsync(dbest, &init, sizeof init, cudaMemcpyHostToDevice, s));
            min_deg_id<<<grid_for(nlast), 256, 0, s>>>(nlast, last, deg, dbest);
            unsigned long long best = 0;
            RCM_CHECK(cudaMemcpyAsync(&best, dbest, sizeof best, cudaMemcpyDeviceToHost, s));
            RCM_CHECK(cudaStreamSynchronize(s));
            node = (int32_t)(best & 0xffffffffu);
        }
    };

    int64_t placed = 0;  // vertices in `order`
    int32_t v = 0;
    while (placed < N) {
        // the smallest unseen vertex (components by ascending smallest id, rcm_permutation :132-134)
        int32_t found = INT32_MAX;
        for (int32_t lo = v; lo < N && found == INT32_MAX; lo = (int32_t)std::min<int64_t>(N, (int64_t)lo + (1 << 22))) {
            const int32_t hi = (int32_t)std::min<int64_t>(N, (int64_t)lo + (1 << 22));
            const int32_t init = INT32_MAX;
            RCM_CHECK(cudaMemcpyAsync(dscal, &init, sizeof init, cudaMemcpyHostToDevice, s));
            first_unseen<<<grid_for(hi - lo), 256, 0, s>>>(lo, hi, seen, dscal);
            RCM_CHECK(cudaMemcpyAsync(&found, dscal, sizeof found, cudaMemcpyDeviceToHost, s));
            RCM_CHECK(cudaStreamSynchronize(s));
        }
        if (found == INT32_MAX) raise(CF_INVALID_ARG, "rcm: vertex accounting");
        v = found;
        int32_t root;
        int32_t in_seen = 1;
        if (seed >= 0 && seed < N) {
            RCM_CHECK(cudaMemcpyAsync(&in_seen, seen + seed, sizeof in_seen, cudaMemcpyDeviceToHost, s));
            RCM_CHECK(cudaStreamSynchronize(s));
        }
        if (seed >= 0 && seed < N && !in_seen) {
            // the seed is used if it lives in this (unvisited) component
            int32_t* last = nullptr;
            int32_t nlast = 0;
            bfs_sets(v, last, nlast);
            int32_t ds = -1;
            RCM_CHECK(cudaMemcpyAsync(&ds, dist + seed, sizeof ds, cudaMemcpyDeviceToHost, s));
            RCM_CHECK(cudaStreamSynchronize(s));
            root = ds >= 0 ? seed : pseudo_peripheral(v);
        } else {
            root = pseudo_peripheral(v);
        }
        // bfs_levels reorder.hpp:54-88, level-synchronous
        const int32_t one = 1;
        RCM_CHECK(cudaMemcpyAsync(seen + root, &one, sizeof one, cudaMemcpyHostToDevice, s));
        RCM_CHECK(cudaMemcpyAsync(order + placed, &root, sizeof root, cudaMemcpyHostToDevice, s));
        int64_t ls = placed, le = placed + 1;
        for (;;) {
            const int32_t nf = (int32_t)(le - ls);
            const int32_t* front = order + ls;
            cm_claim<<<grid_for(nf), 256, 0, s>>>(nf, front, goff, adj, seen, claim);
            cm_count<<<grid_for(nf), 256, 0, s>>>(nf, front, goff, adj, seen, claim, cnt);
            exclusive_scan<int32_t>(cnt, nf, loff, s, ws);
            int64_t tot = 0;
            RCM_CHECK(cudaMemcpyAsync(&tot, loff + nf, sizeof tot, cudaMemcpyDeviceToHost, s));
            RCM_CHECK(cudaStreamSynchronize(s));
            if (tot == 0) break;
            cm_emit<<<grid_for(nf), 256, 0, s>>>(nf, front, goff, adj, deg, seen, claim, loff, order + le);
            RCM_CHECK(cudaGetLastError());
            ls = le;
            le += tot;
        }
        placed = le;
    }
    reverse_labels<<<grid_for(N), 256, 0, s>>>(N, order, new_of_old);
    RCM_CHECK(cudaGetLastError());
    RCM_CHECK(cudaStreamSynchronize(s));
}

std::vector<int32_t> rcm_permutation_device(int32_t N, int64_t E, const int32_t* tets_host, int32_t seed, int device) {
    std::vector<int32_t> new_of_old(N);
    if (N == 0) return new_of_old;
    RCM_CHECK(cudaSetDevice(device));
    cudaStream_t s;
    RCM_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    DevBuf B;
    int32_t* tets = B.alloc<int32_t>(4 * (size_t)E);
    RCM_CHECK(cudaMemcpyAsync(tets, tets_host, 4 * (size_t)E * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    int32_t* labels = B.alloc<int32_t>(N);
    rcm_labels_device(N, E, tets, seed, s, labels);
    B.free(tets);
    RCM_CHECK(cudaMemcpyAsync(new_of_old.data(), labels, (size_t)N * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RCM_CHECK(cudaStreamSynchronize(s));
    return new_of_old;
}

}  // namespace cfb
