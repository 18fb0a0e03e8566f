// cf_tilepack.hpp — per-tile plan construction shared by the host plan builder (cf_plan.cpp)
// and the device setup pipeline (cf_devplan.cu): one implementation, so the two builders
// cannot disagree. Plain __host__ __device__ code over caller-provided workspace (no
// allocation): the host runs one tile per OpenMP iteration, the device one tile per thread.
//
// Reference semantics (paths relative to /root/reference/proj/include/castfem/): a tile is a
// BlockPlan block (blocked.hpp:79-93, 217-307): block-local slots of the nodes its elements
// touch, facet bindings in element order then facet id (blocked.hpp:244-288), per-slot
// contributions summed in ascending element order, then facets (assemble_blocks :454-498).
#pragma once

#include <cmath>
#include <cstdint>

#include "cf_tileblob.hpp"

namespace cfb {

// read-only inputs of the per-tile functions (host or device pointers, all indexed globally
// unless noted)
struct TileCtx {
    const int32_t* tets = nullptr;         // [4E] oriented (finalize_mesh), global node ids
    const int32_t* region = nullptr;       // [E]
    const int32_t* facets = nullptr;       // [3F] global node ids
    const double* coords = nullptr;        // [3N] global
    const int32_t* fe_off = nullptr;       // [E+1] facet bindings per element (ascending facet id)
    const int32_t* fe = nullptr;           // facet ids
    const int32_t* facet_kind = nullptr;   // [F] kind id (>= 0 here: Dirichlet facets are not bound)
    const int32_t* facet_sister = nullptr; // [F] sister element of an interface facet, else -1
    const int32_t* local_of = nullptr;     // [N] global -> local node id (ghosts: >= n_local)
    const uint8_t* lnode_region = nullptr; // [n_local]
    const int8_t* lnode_dir = nullptr;     // [n_local] Dirichlet id or -1; null: none
    const int32_t* ntiles_of = nullptr;    // [n_local] tiles touching the node (pack only)
    const uint8_t* shared_node = nullptr;  // [n_local] rank-shared (multi-rank); null: none
    const uint8_t* kind_interface = nullptr;  // [kinds] 1: interface facet kind
    bool tdep = false, coords_layout = false;
    bool slot_banks = true;                // bank-aware private slot numbering (stored layout)
    bool slot_by_node = true;              // shared slots by node id after the private ones
    int bank_passes = 0;                   // in-block colour swap passes (CF_BANK_PASSES)
    int bank_iters = 0;                    // seeded swap attempts per element (CF_BANK_ITERS)
};

// capacities of one tile's workspace (upper bounds over the tiles it serves)
struct TileCaps {
    int32_t ne, ns, nf, ncsr;
};

CF_HD int64_t tile_ws_ints(const TileCaps& c) {
    const int64_t ne8 = cf_round(c.ne, 8), E4 = 4 * ne8, ng = 4 * (ne8 / 8);
    const int64_t na = c.ncsr + 8;  // phase-3 groups: at most one per padded entry
    return 2 * E4                    // corner ids + sort temp
           + 6 * (int64_t)c.ns + 8   // unique / count / order / slot map pairs (+ temp)
           + E4 + ng + 1             // corner-gather groups (gmem, goff)
           + 2 * ((int64_t)c.ns + 1) + E4  // private slot -> groups CSR (+ cursor)
           + 8 * ng                  // per-group bank counts of fixed slots
           + 3 * (int64_t)c.ns       // ord, bank_of, newtn
           + c.nf                    // tile facets
           + 3 * ((int64_t)c.ns + 1) + E4 + 3 * (int64_t)c.nf  // ent_off, cur, poff, ent
           + c.ncsr + 8              // items
           + 2 * (int64_t)c.ns       // sperm (+ temp)
           + E4                      // eslot
           + 2 * ne8                 // pos, at
           + 2 * (na + 1) + c.ncsr + 8   // a_off, a_items
           + ne8 + 1 + E4            // g_off, g_list
           + 8 * na                  // cnt
           + 64;
}

namespace tp {

// stable bottom-up merge sort of a[0, n) with temp t[0, n) by less(x, y); result in a
template <class T, class L>
CF_HD void merge_sort(T* a, T* t, int n, L less) {
    T* src = a;
    T* dst = t;
    for (int w = 1; w < n; w *= 2) {
        for (int lo = 0; lo < n; lo += 2 * w) {
            const int mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            int i = lo, j = mid, k = lo;
            while (i < mid && j < hi) dst[k++] = less(src[j], src[i]) ? src[j++] : src[i++];
            while (i < mid) dst[k++] = src[i++];
            while (j < hi) dst[k++] = src[j++];
        }
        T* x = src;
        src = dst;
        dst = x;
    }
    if (src != a)
        for (int i = 0; i < n; ++i) a[i] = src[i];
}

// index of v in the ascending array a[0, n) (present by construction)
CF_HD int find_sorted(const int32_t* a, int n, int32_t v) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

// triangle_area geometry.hpp (bitwise the host's: same operation order, no contraction)
CF_HD double tri_area(const double* a, const double* b, const double* c) {
    const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
    const double x[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    return 0.5 * sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
}

struct Bump {  // linear workspace carve-out
    int32_t* p;
    CF_HD int32_t* take(int64_t n) {
        int32_t* r = p;
        p += n;
        return r;
    }
};

}  // namespace tp

// Pass 1 of a tile (elements te[0, ne), ascending global id): its unique local nodes ordered by
// contribution count (descending), then local id -- the warps of the reduction phase then walk
// lists of near-equal length -- and its metadata (ne, ns, nf, ncsr: lists padded to 4).
// tnodes: [ns] out. Returns the metadata.
CF_HD TileMeta tile_pass1(const TileCtx& c, const int32_t* te, int ne, int32_t* tnodes, int32_t* ws) {
    tp::Bump W{ws};
    const int n4 = 4 * ne;
    int32_t* buf = W.take(n4);
    int32_t* tmp = W.take(n4);
    for (int i = 0; i < ne; ++i)
        for (int a = 0; a < 4; ++a) buf[4 * i + a] = c.local_of[c.tets[4 * (int64_t)te[i] + a]];
    tp::merge_sort(buf, tmp, n4, [](int32_t x, int32_t y) { return x < y; });
    int ns = 0;
    int32_t* cnt = tmp;  // reuse: counts per unique node
    for (int k = 0; k < n4; ++k) {
        if (k == 0 || buf[k] != buf[k - 1]) {
            buf[ns] = buf[k];
            cnt[ns] = 0;
            ++ns;
        }
        cnt[ns - 1]++;
    }
    int nf = 0;
    for (int i = 0; i < ne; ++i)
        for (int32_t j = c.fe_off[te[i]]; j < c.fe_off[te[i] + 1]; ++j, ++nf)
            for (int a = 0; a < 3; ++a) cnt[tp::find_sorted(buf, ns, c.local_of[c.facets[3 * (int64_t)c.fe[j] + a]])]++;
    int ncsr = 0;
    for (int k = 0; k < ns; ++k) ncsr += (cnt[k] + 3) & ~3;
    // (count desc, local id asc): a stable sort by count of the ascending unique list
    int32_t* idx = W.take(ns);
    int32_t* it = W.take(ns);
    for (int k = 0; k < ns; ++k) idx[k] = k;
    tp::merge_sort(idx, it, ns, [cnt](int32_t x, int32_t y) { return cnt[x] > cnt[y]; });
    for (int k = 0; k < ns; ++k) tnodes[k] = buf[idx[k]];
    return TileMeta{ne, ns, nf, ncsr};
}

// Footprint of a chunk of elements (global node ids; no local numbering yet): shared-memory
// bytes of its tile (the budget split of build_rank_plan). ws: tile_ws_ints of the chunk.
CF_HD int64_t tile_footprint(const TileCtx& c, const int32_t* te, int ne, int32_t* ws) {
    tp::Bump W{ws};
    const int n4 = 4 * ne;
    int32_t* buf = W.take(n4);
    int32_t* tmp = W.take(n4);
    for (int i = 0; i < ne; ++i)
        for (int a = 0; a < 4; ++a) buf[4 * i + a] = c.tets[4 * (int64_t)te[i] + a];
    tp::merge_sort(buf, tmp, n4, [](int32_t x, int32_t y) { return x < y; });
    int ns = 0;
    int32_t* cnt = tmp;
    for (int k = 0; k < n4; ++k) {
        if (k == 0 || buf[k] != buf[k - 1]) {
            buf[ns] = buf[k];
            cnt[ns] = 0;
            ++ns;
        }
        cnt[ns - 1]++;
    }
    int nf = 0;
    for (int i = 0; i < ne; ++i)
        for (int32_t j = c.fe_off[te[i]]; j < c.fe_off[te[i] + 1]; ++j, ++nf)
            for (int a = 0; a < 3; ++a) cnt[tp::find_sorted(buf, ns, c.facets[3 * (int64_t)c.fe[j] + a])]++;
    int ncsr = 0;
    for (int k = 0; k < ns; ++k) ncsr += (cnt[k] + 3) & ~3;
    const TileLayout L(TileMeta{ne, ns, nf, ncsr}, c.tdep, c.coords_layout);
    return cf_round(L.bytes, 16) + 24 * cf_round(ns, 2) + 8 * cf_round(L.scratch, 2);
}

// Bank-aware local element positions (see cf_plan.cpp's description): the element positions
// inside a tile are a free permutation (the reduction order is fixed by the lists); blocks of 8
// reference-order elements take the 8 bank groups (position & 7) greedily against the
// reduction-read groups of phase 3.
struct BankPlan {
    int ne = 0, ns = 0, na = 0;
    int32_t *pos = nullptr, *at = nullptr;        // element -> position, position -> element
    int32_t *a_off = nullptr, *a_items = nullptr; // phase-3 groups
    int32_t *g_off = nullptr, *g_list = nullptr;  // element -> its phase-3 groups
    int32_t* cnt = nullptr;                       // [8 na] bank load per group
    const int32_t* eslot = nullptr;

    CF_HD int cost_a(int g) const {
        int cn[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t fixed[8];
        int nfix = 0;
        for (int k = a_off[g]; k < a_off[g + 1]; ++k) {
            const uint32_t it = (uint32_t)a_items[k];
            if (it & 0x80000000u) {
                const uint32_t ad = it & 0x7fffffffu;
                bool dup = false;
                for (int f = 0; f < nfix; ++f) dup = dup || fixed[f] == ad;
                if (dup) continue;
                if (nfix < 8) fixed[nfix++] = ad;
                cn[ad & 7]++;
            } else {
                cn[pos[it >> 2] & 7]++;
            }
        }
        int mx = 0;
        for (int b = 0; b < 8; ++b) mx = mx > cn[b] ? mx : cn[b];
        return mx;
    }
    CF_HD int cost_b(int blk, int q) const {
        int cn[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int32_t seen[8];
        int nsn = 0;
        const int end = ne < 8 * blk + 8 ? ne : 8 * blk + 8;
        for (int p = 8 * blk; p < end; ++p) {
            const int32_t sl = eslot[4 * at[p] + q];
            bool dup = false;
            for (int k = 0; k < nsn; ++k) dup = dup || seen[k] == sl;
            if (dup) continue;
            seen[nsn++] = sl;
            cn[sl & 7]++;
        }
        int mx = 0;
        for (int b = 0; b < 8; ++b) mx = mx > cn[b] ? mx : cn[b];
        return mx;
    }
    CF_HD int gmax(int g) const {
        const int32_t* cg = cnt + 8 * (int64_t)g;
        int mx = 0;
        for (int u = 0; u < 8; ++u) mx = mx > cg[u] ? mx : cg[u];
        return mx;
    }
    // items: per slot [off[s], off[s+1]) in reduction order (padded to multiples of 4)
    CF_HD void run(int ne_, int ns_, const int32_t* eslot_, const int32_t* off, const uint32_t* items,
                   const int32_t* sperm, int iters, uint64_t seed, bool greedy, int passes, tp::Bump& W) {
        ne = ne_;
        ns = ns_;
        eslot = eslot_;
        pos = W.take(ne + 8);
        at = W.take(ne + 8);
        for (int i = 0; i < ne; ++i) pos[i] = at[i] = i;
        if (ne < 16) return;
        // phase-3 groups: quarter warps of slots (thread order sperm) x list index
        a_off = W.p;
        a_off[0] = 0;
        na = 0;
        int64_t nitems = 0;
        for (int q0 = 0; q0 < ns; q0 += 8) {
            const int q1 = ns < q0 + 8 ? ns : q0 + 8;
            int mx = 0;
            for (int u = q0; u < q1; ++u) {
                const int l = off[sperm[u] + 1] - off[sperm[u]];
                mx = mx > l ? mx : l;
            }
            for (int j = 0; j < mx; ++j) {
                for (int u = q0; u < q1; ++u)
                    if (off[sperm[u]] + j < off[sperm[u] + 1]) ++nitems;
                a_off[++na] = (int32_t)nitems;
            }
        }
        W.p += na + 1;
        a_items = W.take(nitems);
        {
            int64_t k = 0;
            for (int q0 = 0; q0 < ns; q0 += 8) {
                const int q1 = ns < q0 + 8 ? ns : q0 + 8;
                int mx = 0;
                for (int u = q0; u < q1; ++u) {
                    const int l = off[sperm[u] + 1] - off[sperm[u]];
                    mx = mx > l ? mx : l;
                }
                for (int j = 0; j < mx; ++j)
                    for (int u = q0; u < q1; ++u) {
                        const int sl = sperm[u];
                        if (off[sl] + j < off[sl + 1]) a_items[k++] = (int32_t)items[off[sl] + j];
                    }
            }
        }
        g_off = W.take(ne + 1);
        for (int i = 0; i <= ne; ++i) g_off[i] = 0;
        for (int g = 0; g < na; ++g)
            for (int k = a_off[g]; k < a_off[g + 1]; ++k)
                if (!((uint32_t)a_items[k] & 0x80000000u)) g_off[((uint32_t)a_items[k] >> 2) + 1]++;
        for (int i = 0; i < ne; ++i) g_off[i + 1] += g_off[i];
        g_list = W.take(g_off[ne]);
        {
            int32_t* cur = W.p;  // transient
            for (int i = 0; i < ne; ++i) cur[i] = g_off[i];
            for (int g = 0; g < na; ++g)
                for (int k = a_off[g]; k < a_off[g + 1]; ++k)
                    if (!((uint32_t)a_items[k] & 0x80000000u)) g_list[cur[(uint32_t)a_items[k] >> 2]++] = g;
        }
        cnt = W.take(8 * (int64_t)na);
        if (greedy) {
            for (int64_t k = 0; k < 8 * (int64_t)na; ++k) cnt[k] = 0;
            for (int g = 0; g < na; ++g) {
                uint32_t fixed[64];
                int nfix = 0;
                for (int k = a_off[g]; k < a_off[g + 1]; ++k) {
                    const uint32_t it = (uint32_t)a_items[k];
                    if (!(it & 0x80000000u)) continue;
                    const uint32_t ad = it & 0x7fffffffu;
                    bool dup = false;
                    for (int f = 0; f < nfix; ++f) dup = dup || fixed[f] == ad;
                    if (dup) continue;
                    if (nfix < 64) fixed[nfix++] = ad;
                    cnt[8 * (int64_t)g + (ad & 7)]++;
                }
            }
            // blocks of 8 consecutive elements take the 8 colours as a permutation; score: added
            // wavefronts (a count reaching its group's maximum), then load
            for (int b0 = 0; b0 < ne; b0 += 8) {
                const int nb = ne - b0 < 8 ? ne - b0 : 8;
                bool used[8] = {false, false, false, false, false, false, false, false};
                for (int i = b0; i < b0 + nb; ++i) {
                    int best = -1, best_score = 1 << 30;
                    for (int cc = 0; cc < nb; ++cc) {
                        if (used[cc]) continue;
                        int sc = 0;
                        for (int k = g_off[i]; k < g_off[i + 1]; ++k) {
                            const int32_t* cg = cnt + 8 * (int64_t)g_list[k];
                            int mx = 0;
                            for (int u = 0; u < 8; ++u) mx = mx > cg[u] ? mx : cg[u];
                            sc += 64 * (cg[cc] + 1 > mx) + cg[cc];
                        }
                        if (sc < best_score) {
                            best_score = sc;
                            best = cc;
                        }
                    }
                    used[best] = true;
                    for (int k = g_off[i]; k < g_off[i + 1]; ++k) cnt[8 * (int64_t)g_list[k] + best]++;
                    pos[i] = b0 + best;
                    at[b0 + best] = i;
                }
            }
            // optional pairwise colour swaps inside a block while they lower the reduction reads
            int touched[16];
            for (int pass = 0; pass < passes; ++pass) {
                bool improved = false;
                for (int b0 = 0; b0 < ne; b0 += 8) {
                    const int nb = ne - b0 < 8 ? ne - b0 : 8;
                    for (int u = 0; u < nb; ++u)
                        for (int v = u + 1; v < nb; ++v) {
                            const int i1 = at[b0 + u], i2 = at[b0 + v];
                            const int c1 = pos[i1] & 7, c2 = pos[i2] & 7;
                            int nt = 0;
                            const int ii[2] = {i1, i2};
                            for (int w = 0; w < 2; ++w)
                                for (int k = g_off[ii[w]]; k < g_off[ii[w] + 1]; ++k) {
                                    bool dup = false;
                                    for (int z = 0; z < nt; ++z) dup = dup || touched[z] == g_list[k];
                                    if (!dup && nt < 16) touched[nt++] = g_list[k];
                                }
                            int before = 0;
                            for (int z = 0; z < nt; ++z) before += gmax(touched[z]);
                            auto move = [&](int i, int from, int to) {
                                for (int k = g_off[i]; k < g_off[i + 1]; ++k) {
                                    cnt[8 * (int64_t)g_list[k] + from]--;
                                    cnt[8 * (int64_t)g_list[k] + to]++;
                                }
                            };
                            move(i1, c1, c2);
                            move(i2, c2, c1);
                            int after = 0;
                            for (int z = 0; z < nt; ++z) after += gmax(touched[z]);
                            if (after < before) {
                                pos[i1] = b0 + c2;
                                pos[i2] = b0 + c1;
                                at[b0 + c2] = i1;
                                at[b0 + c1] = i2;
                                improved = true;
                            } else {
                                move(i1, c2, c1);
                                move(i2, c1, c2);
                            }
                        }
                }
                if (!improved) break;
            }
        }
        uint64_t x = seed * 0x9E3779B97F4A7C15ull + 0x2545F4914F6CDD1Dull;
        int ga[16], gb[2];
        for (int it = 0; it < iters; ++it) {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            const int i1 = (int)(x % (uint64_t)ne);
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            const int i2 = (int)(x % (uint64_t)ne);
            const int p1 = pos[i1], p2 = pos[i2];
            if ((p1 & 7) == (p2 & 7) && (p1 >> 3) == (p2 >> 3)) continue;
            int nga = 0;
            const int ii[2] = {i1, i2};
            for (int w = 0; w < 2; ++w)
                for (int k = g_off[ii[w]]; k < g_off[ii[w] + 1]; ++k) {
                    bool dup = false;
                    for (int u = 0; u < nga; ++u) dup = dup || ga[u] == g_list[k];
                    if (!dup && nga < 16) ga[nga++] = g_list[k];
                }
            const int nb = (p1 >> 3) == (p2 >> 3) ? 1 : 2;
            gb[0] = p1 >> 3;
            gb[1] = p2 >> 3;
            auto total = [&]() {
                int cc = 0;
                for (int u = 0; u < nga; ++u) cc += cost_a(ga[u]);
                for (int u = 0; u < nb; ++u)
                    for (int q = 0; q < 4; ++q) cc += cost_b(gb[u], q);
                return cc;
            };
            const int before = total();
            int32_t s_ = pos[i1];
            pos[i1] = pos[i2];
            pos[i2] = s_;
            at[p1] = i2;
            at[p2] = i1;
            if (total() > before) {
                s_ = pos[i1];
                pos[i1] = pos[i2];
                pos[i2] = s_;
                at[p1] = i1;
                at[p2] = i2;
            }
        }
    }
    CF_HD int64_t total_cost(int which = 3) const {  // 1: phase-3 reads, 2: phase-2a gathers
        int64_t cc = 0;
        if (ne < 16) return 0;
        if (which & 1)
            for (int g = 0; g < na; ++g) cc += cost_a(g);
        if (which & 2)
            for (int b = 0; 8 * b < ne; ++b)
                for (int q = 0; q < 4; ++q) cc += cost_b(b, q);
        return cc;
    }
};

// outputs of one tile's packing
struct TileOut {
    uint8_t* stg = nullptr;          // the tile's [conn, bytes) sections (zeroed by the caller)
    int32_t* elem_global = nullptr;  // [ne] global element id at each local position
    int32_t* tets_ord = nullptr;     // [4 ne] local node ids at each position (null: not wanted)
    int32_t* slot_node = nullptr;    // [round2(ns)] (region << 28 | local id), padding -1
    int32_t n_if = 0, n_bc = 0;
    int64_t bank_cost[3] = {0, 0, 0};  // diagnostics (want_cost): all, reduction reads, gathers
};

// Packs one tile: slot order (tile-private first by contribution count, then the tile-shared
// nodes by node id), bank-aware private slot numbering, per-slot contribution lists in
// reduction order (ascending element, then facets; padded to 4 with the zero operand),
// reduction thread order, bank-aware element positions, and every non-geometry section of the
// blob. tnodes: pass 1's order (count desc, local id asc), ns entries.
CF_HD void tile_pack(const TileCtx& c, int32_t tile, const int32_t* te, const TileMeta& tm, const int32_t* tnodes,
                     int32_t* ws, TileOut& out, bool want_cost = false) {
    const TileLayout L(tm, c.tdep, c.coords_layout);
    const int ne = tm.ne, ns = tm.ns, nf = tm.nf;
    const int ne8 = (int)cf_round(ne, 8);
    tp::Bump W{ws};
    int32_t* tn = W.take(ns);
    auto priv = [&](int32_t l) { return c.ntiles_of[l] == 1 && !(c.shared_node && c.shared_node[l]); };
    // slot order: stable partition (private first), shared ascending by node id
    int np = 0;
    if (c.slot_by_node) {
        for (int k = 0; k < ns; ++k)
            if (priv(tnodes[k])) tn[np++] = tnodes[k];
        int q = np;
        for (int k = 0; k < ns; ++k)
            if (!priv(tnodes[k])) tn[q++] = tnodes[k];
        int32_t* tmp = W.take(ns);
        tp::merge_sort(tn + np, tmp, ns - np, [](int32_t x, int32_t y) { return x < y; });
    } else {
        for (int k = 0; k < ns; ++k) tn[k] = tnodes[k];
        W.take(ns);
        while (np < ns && priv(tn[np])) ++np;
    }
    // slot lookup: (local id, slot) sorted by local id
    int32_t* key = W.take(ns);
    int32_t* sl_of = W.take(ns);
    auto build_lookup = [&]() {
        int32_t* tmpk = W.p;  // transient scratch after the live carve-outs
        for (int k = 0; k < ns; ++k) tmpk[k] = k;
        int32_t* tmpi = tmpk + ns;
        tp::merge_sort(tmpk, tmpi, ns, [&](int32_t x, int32_t y) { return tn[x] < tn[y]; });
        for (int k = 0; k < ns; ++k) {
            key[k] = tn[tmpk[k]];
            sl_of[k] = tmpk[k];
        }
    };
    build_lookup();
    auto slot = [&](int32_t l) { return sl_of[tp::find_sorted(key, ns, l)]; };
    // bank-aware numbering of the tile-private slots (their order is free): spread each block of
    // 8 consecutive elements' corner-q slots over the 8 bank groups (slot & 7); shared slots fixed
    if (!c.coords_layout && ne >= 16 && c.slot_banks && c.slot_by_node) {
        // np counted as the private prefix, like the host's scan of the partitioned order
        if (np >= 16) {
            const int ng = 4 * ((ne + 7) / 8);
            int32_t* goff = W.take(ng + 1);
            int32_t* gmem = W.take(4 * (int64_t)ne8);
            goff[0] = 0;
            int n_gm = 0;
            for (int b0 = 0, g = 0; b0 < ne; b0 += 8)
                for (int q = 0; q < 4; ++q, ++g) {
                    const int end = ne < b0 + 8 ? ne : b0 + 8;
                    for (int i = b0; i < end; ++i) {
                        const int32_t s = slot(c.local_of[c.tets[4 * (int64_t)te[i] + q]]);
                        bool dup = false;
                        for (int k = goff[g]; k < n_gm; ++k) dup = dup || gmem[k] == s;
                        if (!dup) gmem[n_gm++] = s;
                    }
                    goff[g + 1] = n_gm;
                }
            // private slot (old index) -> its groups (CSR in group order)
            int32_t* pgo = W.take(np + 1);
            int32_t* pgc = W.take(np + 1);
            for (int k = 0; k <= np; ++k) pgo[k] = 0;
            for (int g = 0; g < ng; ++g)
                for (int k = goff[g]; k < goff[g + 1]; ++k)
                    if (gmem[k] < np) pgo[gmem[k] + 1]++;
            for (int k = 0; k < np; ++k) pgo[k + 1] += pgo[k];
            int32_t* pgl = W.take(pgo[np]);
            for (int k = 0; k < np; ++k) pgc[k] = pgo[k];
            for (int g = 0; g < ng; ++g)
                for (int k = goff[g]; k < goff[g + 1]; ++k)
                    if (gmem[k] < np) pgl[pgc[gmem[k]]++] = g;
            int32_t* gcnt = W.take(8 * (int64_t)ng);
            for (int64_t k = 0; k < 8 * (int64_t)ng; ++k) gcnt[k] = 0;
            for (int g = 0; g < ng; ++g)
                for (int k = goff[g]; k < goff[g + 1]; ++k)
                    if (gmem[k] >= np) gcnt[8 * (int64_t)g + (gmem[k] & 7)]++;
            int freeb[8];
            for (int b = 0; b < 8; ++b) freeb[b] = (np - b + 7) / 8;
            int32_t* ord = W.take(np);
            int32_t* otmp = W.take(np);
            for (int k = 0; k < np; ++k) ord[k] = k;
            tp::merge_sort(ord, otmp, np,
                           [&](int32_t x, int32_t y) { return pgo[x + 1] - pgo[x] > pgo[y + 1] - pgo[y]; });
            int32_t* bank_of = otmp;
            for (int w = 0; w < np; ++w) {
                const int32_t o = ord[w];
                int best = -1, bc = 1 << 30;
                for (int b = 0; b < 8; ++b) {
                    if (!freeb[b]) continue;
                    int cc = 0;
                    for (int k = pgo[o]; k < pgo[o + 1]; ++k) cc += gcnt[8 * (int64_t)pgl[k] + b];
                    if (cc < bc || (cc == bc && freeb[b] > freeb[best])) {
                        bc = cc;
                        best = b;
                    }
                }
                bank_of[o] = best;
                freeb[best]--;
                for (int k = pgo[o]; k < pgo[o + 1]; ++k) gcnt[8 * (int64_t)pgl[k] + best]++;
            }
            // new index: the k-th private slot of bank b gets b + 8k (stable in old order)
            int nextb[8];
            for (int b = 0; b < 8; ++b) nextb[b] = b;
            int32_t* newtn = ord;  // ord no longer needed
            for (int o = 0; o < np; ++o) {
                newtn[nextb[bank_of[o]]] = tn[o];
                nextb[bank_of[o]] += 8;
            }
            for (int k = 0; k < np; ++k) tn[k] = newtn[k];
            W.p = goff;  // release the transient carve-outs
            build_lookup();
        }
    }
    // tile facets: element order, then facet id
    int32_t* tf = W.take(nf + 1);
    {
        int k = 0;
        for (int i = 0; i < ne; ++i)
            for (int32_t j = c.fe_off[te[i]]; j < c.fe_off[te[i] + 1]; ++j) tf[k++] = c.fe[j];
    }
    // per-slot contributions in reduction order: element corner (i << 2 | q), or
    // 0x80000000 | the final 16-bit code of a facet term
    int32_t* eslot = W.take(4 * (int64_t)ne8);
    for (int i = 0; i < ne; ++i)
        for (int a = 0; a < 4; ++a) eslot[4 * i + a] = slot(c.local_of[c.tets[4 * (int64_t)te[i] + a]]);
    int32_t* fslot = W.take(3 * (int64_t)nf + 1);
    for (int i = 0; i < nf; ++i)
        for (int a = 0; a < 3; ++a) fslot[3 * i + a] = slot(c.local_of[c.facets[3 * (int64_t)tf[i] + a]]);
    int32_t* ent_off = W.take(ns + 1);
    for (int k = 0; k <= ns; ++k) ent_off[k] = 0;
    for (int k = 0; k < 4 * ne; ++k) ent_off[eslot[k] + 1]++;
    for (int k = 0; k < 3 * nf; ++k) ent_off[fslot[k] + 1]++;
    for (int k = 0; k < ns; ++k) ent_off[k + 1] += ent_off[k];
    uint32_t* ent = (uint32_t*)W.take(ent_off[ns]);
    {
        int32_t* cur = W.p;  // transient
        for (int k = 0; k < ns; ++k) cur[k] = ent_off[k];
        for (int i = 0; i < ne; ++i)
            for (int a = 0; a < 4; ++a) ent[cur[eslot[4 * i + a]]++] = (uint32_t)(i << 2 | a);
        for (int i = 0; i < nf; ++i)
            for (int a = 0; a < 3; ++a) ent[cur[fslot[3 * i + a]]++] = 0x80000000u | L.code_facet(i, a);
    }
    int32_t* poff = W.take(ns + 1);
    poff[0] = 0;
    for (int k = 0; k < ns; ++k) poff[k + 1] = poff[k] + ((ent_off[k + 1] - ent_off[k] + 3) & ~3);
    uint32_t* items = (uint32_t*)W.take(poff[ns]);
    for (int32_t q = 0; q < poff[ns]; ++q) items[q] = 0x80000000u | L.code_zero();
    for (int k = 0; k < ns; ++k)
        for (int32_t q = ent_off[k]; q < ent_off[k + 1]; ++q) items[poff[k] + (q - ent_off[k])] = ent[q];
    // phase-3 thread order: slots by padded list length (descending), stable
    int32_t* sperm = W.take(ns);
    {
        int32_t* t2 = W.take(ns);
        for (int k = 0; k < ns; ++k) sperm[k] = k;
        tp::merge_sort(sperm, t2, ns,
                       [poff](int32_t x, int32_t y) { return poff[x + 1] - poff[x] > poff[y + 1] - poff[y]; });
    }
    BankPlan bank;
    bank.run(ne, ns, eslot, poff, items, sperm, c.coords_layout ? 0 : c.bank_iters * ne, (uint64_t)tile + 1, true,
             c.bank_passes, W);
    if (want_cost && !c.coords_layout) {
        out.bank_cost[0] = bank.total_cost();
        out.bank_cost[1] = bank.total_cost(1);
        out.bank_cost[2] = bank.total_cost(2);
    }
    const int32_t* lp = bank.pos;  // element i -> local position
    uint8_t* stg = out.stg;
    auto at = [&](int32_t off) { return stg + L.stage_of(off); };
    uint16_t* csec = (uint16_t*)at(L.conn);
    for (int i = 0; i < ne; ++i) {
        const int32_t e = te[i], p = lp[i];
        out.elem_global[p] = e;
        for (int a = 0; a < 4; ++a) {
            if (out.tets_ord) out.tets_ord[4 * p + a] = c.local_of[c.tets[4 * (int64_t)e + a]];
            csec[4 * p + a] = (uint16_t)eslot[4 * i + a];
        }
        *at(L.region + p) = (uint8_t)c.region[e];
    }
    for (int i = 0; i < nf; ++i) {
        const int32_t f = tf[i];
        const int32_t kind = c.facet_kind[f];
        uint8_t* rec = at(L.fac + 48 * i);  // (area, slots + kind), sister nodes, pad
        uint16_t* fs = (uint16_t*)(rec + 8);
        for (int a = 0; a < 3; ++a) fs[a] = (uint16_t)fslot[3 * i + a];
        fs[3] = (uint16_t)kind;
        const int32_t* fn = c.facets + 3 * (int64_t)f;
        const double area = tp::tri_area(c.coords + 3 * (int64_t)fn[0], c.coords + 3 * (int64_t)fn[1],
                                         c.coords + 3 * (int64_t)fn[2]);
        *(double*)rec = area;
        int32_t* sis = (int32_t*)(rec + 16);
        if (c.kind_interface[kind]) {
            const int32_t se = c.facet_sister[f];
            for (int a = 0; a < 4; ++a) sis[a] = c.local_of[c.tets[4 * (int64_t)se + a]];
            out.n_if++;
        } else {
            out.n_bc++;
        }
    }
    uint16_t* sp = (uint16_t*)at(L.sperm);
    for (int j = 0; j < ns; ++j) sp[j] = (uint16_t)sperm[j];
    uint16_t* cend = (uint16_t*)at(L.csr_end);
    uint16_t* csr = (uint16_t*)at(L.csr);
    int32_t* sn = (int32_t*)at(L.snode);
    const int nsr = (int)cf_round(ns, 2);
    for (int k = 0; k < nsr; ++k) {
        if (k >= ns) {  // padding slot (never a merge target)
            out.slot_node[k] = -1;
            continue;
        }
        const int32_t l = tn[k];
        const uint32_t reg = c.lnode_region[l];
        out.slot_node[k] = (int32_t)((reg << 28) | (uint32_t)l);
        const bool dir = c.lnode_dir && c.lnode_dir[l] >= 0;
        *at(L.sinfo + k) = (uint8_t)((reg & 0x3f) | (dir ? 0x40 : 0) | (priv(l) ? 0x80 : 0));
        for (int32_t q = poff[k]; q < poff[k + 1]; ++q) {
            const uint32_t it = items[q];
            csr[q] = (it & 0x80000000u) ? (uint16_t)(it & 0xffffu) : L.code_elem(lp[it >> 2], (int)(it & 3));
        }
        cend[k] = (uint16_t)poff[k + 1];
        sn[k] = l;
    }
}

}  // namespace cfb
