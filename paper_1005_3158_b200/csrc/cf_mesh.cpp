// cf_mesh.cpp — mesh-side setup of the B200 castfem path (host, C++20, OpenMP).
//
// Restates, for large meshes, the reference's mesh validation, sister
// pairing and RCM (paths relative to /root/reference/proj/include/castfem/):
//   tet_geometry            geometry.hpp:48-77
//   finalize_mesh           mesh.hpp:148-207 (node_regions :129-144)
//   pair_sister_facets      mesh.hpp:456-478 (CentroidIndex :349-449 semantics)
//   build_node_graph        reorder.hpp:17-24
//   rcm_permutation         reorder.hpp:127-148 (bfs_levels :54-88, pseudo_peripheral :91-120)
//   bandwidth               reorder.hpp:41-48
// plus builder-written pieces the reference lacks: RCB partitioning and the
// structured Kuhn fixtures.
#include <omp.h>
#include <parallel/algorithm>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>

#include "cf_internal.hpp"

namespace cfb {

// ------------------------------------------------------------------ geometry
static inline void sub3(const double* a, const double* b, double* r) {
    r[0] = a[0] - b[0];
    r[1] = a[1] - b[1];
    r[2] = a[2] - b[2];
}
static inline double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static inline void cross3(const double* a, const double* b, double* r) {
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
}
static inline double norm3(const double* a) { return std::sqrt(dot3(a, a)); }

bool tet_geometry(const double* p0, const double* p1, const double* p2, const double* p3, Geom& g) {
    double e1[3], e2[3], e3[3], c[3];
    sub3(p1, p0, e1);
    sub3(p2, p0, e2);
    sub3(p3, p0, e3);
    cross3(e2, e3, c);
    const double det = dot3(e1, c);
    g.vol = det / 6.0;
    const double* p[4] = {p0, p1, p2, p3};
    double d[3];
    sub3(p1, p0, d);
    g.min_edge = g.max_edge = norm3(d);
    for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b) {
            sub3(p[b], p[a], d);
            const double len = norm3(d);
            g.min_edge = std::min(g.min_edge, len);
            g.max_edge = std::max(g.max_edge, len);
        }
    const double eps = 1e-12 * g.max_edge * g.max_edge * g.max_edge;
    if (!(g.vol > eps)) return false;
    const double inv = 1.0 / det;
    double t[3];
    cross3(e2, e3, t);
    for (int k = 0; k < 3; ++k) g.g[1][k] = t[k] * inv;
    cross3(e3, e1, t);
    for (int k = 0; k < 3; ++k) g.g[2][k] = t[k] * inv;
    cross3(e1, e2, t);
    for (int k = 0; k < 3; ++k) g.g[3][k] = t[k] * inv;
    for (int k = 0; k < 3; ++k) g.g[0][k] = ((g.g[1][k] + g.g[2][k]) + g.g[3][k]) * -1.0;
    return true;
}

double triangle_area(const double* a, const double* b, const double* c) {
    double u[3], v[3], w[3];
    sub3(b, a, u);
    sub3(c, a, v);
    cross3(u, v, w);
    return 0.5 * norm3(w);
}
void triangle_centroid(const double* a, const double* b, const double* c, double* out) {
    for (int k = 0; k < 3; ++k) out[k] = ((a[k] + b[k]) + c[k]) * (1.0 / 3.0);
}

void trace_stage(const char* name) {
    static const bool on = std::getenv("CF_TRACE_SETUP") && std::atoi(std::getenv("CF_TRACE_SETUP"));
    static auto last = std::chrono::steady_clock::now();
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cf setup] %-24s %8.3f s\n", name, std::chrono::duration<double>(now - last).count());
    last = now;
}

// ------------------------------------------------------------------ finalize
namespace {
struct FaceKey {
    int32_t k[3];
};
inline void sort3(int32_t* k) {
    if (k[0] > k[1]) std::swap(k[0], k[1]);
    if (k[1] > k[2]) std::swap(k[1], k[2]);
    if (k[0] > k[1]) std::swap(k[0], k[1]);
}
inline uint64_t hash3(const int32_t* k) {
    uint64_t h = (uint64_t)(uint32_t)k[0] * 0x9E3779B97F4A7C15ull;
    h ^= ((uint64_t)(uint32_t)k[1] + 0x7F4A7C159E3779B9ull) * 0xBF58476D1CE4E5B9ull;
    h ^= ((uint64_t)(uint32_t)k[2] + 0x94D049BB133111EBull) * 0xC2B2AE3D27D4EB4Full;
    h ^= h >> 29;
    return h;
}
struct FacetHash {
    size_t mask = 0;
    std::vector<int32_t> slot;  // facet id or -1
    std::vector<FaceKey> keys;  // per facet sorted key
    void build(int32_t F, const int32_t* facets) {
        keys.resize(F);
        size_t cap = 16;
        while (cap < 2 * (size_t)F + 16) cap <<= 1;
        mask = cap - 1;
        slot.assign(cap, -1);
        for (int32_t f = 0; f < F; ++f) {
            FaceKey k{{facets[3 * (size_t)f], facets[3 * (size_t)f + 1], facets[3 * (size_t)f + 2]}};
            sort3(k.k);
            keys[f] = k;
            size_t h = hash3(k.k) & mask;
            while (slot[h] >= 0 && std::memcmp(keys[slot[h]].k, k.k, 12) != 0) h = (h + 1) & mask;
            if (slot[h] < 0) slot[h] = f;  // duplicate facets map to the first
        }
    }
    int32_t find(const int32_t* k) const {
        size_t h = hash3(k) & mask;
        while (slot[h] >= 0) {
            if (std::memcmp(keys[slot[h]].k, k, 12) == 0) return slot[h];
            h = (h + 1) & mask;
        }
        return -1;
    }
};
}  // namespace

Geom MeshData::geometry(int64_t e) const {
    Geom g;
    const int32_t* t = &tets[4 * (size_t)e];
    tet_geometry(pos(t[0]), pos(t[1]), pos(t[2]), pos(t[3]), g);
    return g;
}

void finalize_mesh(const cf_mesh_desc* d, MeshData& m) {
    if (!d || d->n_nodes < 0 || d->n_elems < 0 || d->n_facets < 0) raise(CF_INVALID_ARG, "bad mesh descriptor");
    if ((d->n_nodes && !d->coords) || (d->n_elems && (!d->tets || !d->region)) ||
        (d->n_facets && (!d->facets || !d->facet_tag)) || (d->n_tags && !d->tags) ||
        (d->n_contacts && !d->contacts))
        raise(CF_INVALID_ARG, "null array in mesh descriptor");
    m.N = d->n_nodes;
    m.E = d->n_elems;
    m.F = d->n_facets;
    m.coords = d->coords;
    m.region = d->region;
    m.facets = d->facets;
    m.facet_tag = d->facet_tag;
    m.tags.clear();
    for (int32_t t = 0; t < d->n_tags; ++t) m.tags.emplace_back(d->tags[t] ? d->tags[t] : "");
    m.contacts.assign(d->contacts, d->contacts + 2 * (size_t)d->n_contacts);
    const int64_t N = m.N, E = m.E, F = m.F;

    for (int64_t i = 0; i < 3 * N; ++i)
        if (!std::isfinite(d->coords[i])) raise(CF_VALIDATION, "non-finite node coordinate");

    m.tets.resize(4 * (size_t)E);
    std::atomic<int64_t> bad_e{-1};
    int32_t max_region = 0;
    for (int64_t e = 0; e < E; ++e) max_region = std::max(max_region, d->region[e]);
    const int nreg = max_region + 1;
    const int nthr = omp_get_max_threads();
    std::vector<double> tmin((size_t)nthr * nreg, INFINITY);
    std::atomic<int> bad_code{0};
    m.region_count = 0;
    int32_t rc = 0;
#pragma omp parallel reduction(max : rc)
    {
        std::vector<double> loc(nreg, INFINITY);  // per-thread minima (no shared cache lines)
#pragma omp for schedule(static)
        for (int64_t e = 0; e < E; ++e) {
            int32_t* t = &m.tets[4 * (size_t)e];
            int code = 0;
            for (int a = 0; a < 4; ++a) {
                t[a] = d->tets[4 * (size_t)e + a];
                if (t[a] < 0 || t[a] >= N) code = 1;
            }
            if (!code)
                for (int a = 0; a < 4; ++a)
                    for (int b = a + 1; b < 4; ++b)
                        if (t[a] == t[b]) code = 2;
            if (!code && d->region[e] < 0) code = 3;
            if (!code) {
                rc = std::max(rc, d->region[e] + 1);
                const double *p0 = m.pos(t[0]), *p1 = m.pos(t[1]), *p2 = m.pos(t[2]), *p3 = m.pos(t[3]);
                double e1[3], e2[3], e3[3], c[3];
                sub3(p1, p0, e1);
                sub3(p2, p0, e2);
                sub3(p3, p0, e3);
                cross3(e2, e3, c);
                if (dot3(e1, c) / 6.0 < 0) std::swap(t[2], t[3]);  // tet_signed_volume < 0 (mesh.hpp:170-172)
                Geom g;
                if (!tet_geometry(m.pos(t[0]), m.pos(t[1]), m.pos(t[2]), m.pos(t[3]), g)) code = 4;
                double& mn = loc[d->region[e]];
                mn = std::min(mn, g.min_edge);
            }
            if (code) {
                int64_t cur = bad_e.load();
                while ((cur < 0 || e < cur) && !bad_e.compare_exchange_weak(cur, e)) {
                }
                if (bad_e.load() == e) bad_code = code;
            }
        }
        for (int r = 0; r < nreg; ++r) tmin[(size_t)omp_get_thread_num() * nreg + r] = loc[r];
    }
    m.region_count = rc;
    m.region_min_edge.assign(nreg, INFINITY);
    for (int th = 0; th < nthr; ++th)
        for (int r = 0; r < nreg; ++r) m.region_min_edge[r] = std::min(m.region_min_edge[r], tmin[(size_t)th * nreg + r]);
    if (bad_e >= 0) {
        // report the first offending element in element order (serial recheck)
        const int64_t e = bad_e;
        const int32_t* t = &d->tets[4 * (size_t)e];
        for (int a = 0; a < 4; ++a)
            if (t[a] < 0 || t[a] >= N)
                raise(CF_VALIDATION, "element " + std::to_string(e) + " references node " + std::to_string(t[a]) +
                                         " outside [0, " + std::to_string(N) + ")");
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b)
                if (t[a] == t[b])
                    raise(CF_VALIDATION, "element " + std::to_string(e) + " has repeated node " + std::to_string(t[a]));
        if (d->region[e] < 0) raise(CF_VALIDATION, "negative region id");
        Geom g;  // the reference's message (geometry.hpp:66-69, mesh.hpp:175-176)
        const int32_t* to = &m.tets[4 * (size_t)e];
        tet_geometry(m.pos(to[0]), m.pos(to[1]), m.pos(to[2]), m.pos(to[3]), g);
        raise(CF_DEGENERATE, "element " + std::to_string(e) + ": degenerate tetrahedron: volume " +
                                 std::to_string(g.vol) + " below threshold " +
                                 std::to_string(1e-12 * g.max_edge * g.max_edge * g.max_edge));
    }

    trace_stage("finalize: geometry");
    // node_regions (mesh.hpp:129-144): parallel first claim; on a conflict the serial scan
    // reports the reference's first offending (element, node) pair
    m.node_region.assign(N, -1);
    bool conflict = false;
#pragma omp parallel for schedule(static) reduction(|| : conflict)
    for (int64_t e = 0; e < E; ++e)
        for (int a = 0; a < 4; ++a) {
            std::atomic_ref<int32_t> w(m.node_region[m.tets[4 * (size_t)e + a]]);
            int32_t cur = -1;
            if (!w.compare_exchange_strong(cur, d->region[e], std::memory_order_relaxed) && cur != d->region[e])
                conflict = true;
        }
    if (conflict) {
        std::fill(m.node_region.begin(), m.node_region.end(), -1);
        for (int64_t e = 0; e < E; ++e)
            for (int a = 0; a < 4; ++a) {
                const int32_t n = m.tets[4 * (size_t)e + a];
                if (m.node_region[n] >= 0 && m.node_region[n] != d->region[e])
                    raise(CF_VALIDATION, "node " + std::to_string(n) + " belongs to elements of regions " +
                                             std::to_string(m.node_region[n]) + " and " + std::to_string(d->region[e]));
                m.node_region[n] = d->region[e];
            }
    }
    for (int64_t n = 0; n < N; ++n)
        if (m.node_region[n] < 0) raise(CF_VALIDATION, "node " + std::to_string(n) + " not referenced by any element");

    // facet owners (mesh.hpp:182-201): the unique element having the face
    for (int64_t f = 0; f < F; ++f)
        for (int a = 0; a < 3; ++a) {
            const int32_t n = d->facets[3 * (size_t)f + a];
            if (n < 0 || n >= N)
                raise(CF_VALIDATION, "facet " + std::to_string(f) + " references node " + std::to_string(n) +
                                         " outside [0, " + std::to_string(N) + ")");
        }
    trace_stage("finalize: node regions");
    m.owner.assign(F, -1);
    if (F > 0) {
        FacetHash H;
        H.build((int32_t)F, d->facets);
        std::vector<std::atomic<int32_t>> cnt(F);
        std::vector<std::atomic<int32_t>> own(F);
        for (int64_t f = 0; f < F; ++f) {
            cnt[f] = 0;
            own[f] = INT32_MAX;
        }
        static const int tf[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
        // only faces whose three nodes all lie on some facet can match one
        std::vector<uint8_t> on_facet(N, 0);
        for (int64_t i = 0; i < 3 * F; ++i) on_facet[d->facets[i]] = 1;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < E; ++e) {
            const int32_t* t = &m.tets[4 * (size_t)e];
            const int on = on_facet[t[0]] + on_facet[t[1]] + on_facet[t[2]] + on_facet[t[3]];
            if (on < 3) continue;
            for (int j = 0; j < 4; ++j) {
                if (!on_facet[t[tf[j][0]]] || !on_facet[t[tf[j][1]]] || !on_facet[t[tf[j][2]]]) continue;
                int32_t k[3] = {t[tf[j][0]], t[tf[j][1]], t[tf[j][2]]};
                sort3(k);
                const int32_t f = H.find(k);
                if (f < 0) continue;
                cnt[f].fetch_add(1);
                int32_t cur = own[f].load();
                while ((int32_t)e < cur && !own[f].compare_exchange_weak(cur, (int32_t)e)) {
                }
            }
        }
        for (int64_t f = 0; f < F; ++f) {
            const int32_t g = H.find(H.keys[f].k);  // duplicates share the first's counters
            if (cnt[g] == 0) raise(CF_VALIDATION, "facet " + std::to_string(f) + " is not a face of any element");
            if (cnt[g] > 1)
                raise(CF_VALIDATION, "facet " + std::to_string(f) + " is an interior face (two owner elements)");
            m.owner[f] = own[g];
        }
    }
    for (size_t c = 0; c < m.contacts.size(); ++c)
        if (m.contacts[c] < 0 || m.contacts[c] >= (int32_t)m.tags.size())
            raise(CF_VALIDATION, "contact declaration references unknown tag");
    trace_stage("finalize: facet owners");
}

// ------------------------------------------------------------------ sisters
namespace {
struct Cand {
    double c[3];
    int32_t facet, owner;
};
// Exact nearest-centroid index: uniform grid + ring search whose stopping
// bound keeps a full cell of slack, so every candidate tying the best (d2,
// owner, facet) is visited — the CentroidIndex contract (mesh.hpp:347-449).
struct Grid {
    std::vector<Cand> pts;
    double lo[3], cell = 0;
    int64_t dims[3] = {1, 1, 1};
    std::vector<int64_t> off;
    std::vector<int32_t> items;
    void build() {
        for (int k = 0; k < 3; ++k) lo[k] = pts.empty() ? 0 : pts[0].c[k];
        double hi[3] = {lo[0], lo[1], lo[2]};
        for (auto& p : pts)
            for (int k = 0; k < 3; ++k) {
                lo[k] = std::min(lo[k], p.c[k]);
                hi[k] = std::max(hi[k], p.c[k]);
            }
        const double diag = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
        cell = std::max(diag / std::cbrt((double)std::max<size_t>(pts.size(), 1)), diag * 1e-9);
        if (!(cell > 0)) cell = 1.0;
        for (int k = 0; k < 3; ++k) dims[k] = std::min<int64_t>(4096, (int64_t)((hi[k] - lo[k]) / cell) + 1);
        off.assign(dims[0] * dims[1] * dims[2] + 1, 0);
        std::vector<int64_t> cellof(pts.size());
        for (size_t i = 0; i < pts.size(); ++i) {
            cellof[i] = cell_of(pts[i].c);
            off[cellof[i] + 1]++;
        }
        for (size_t i = 1; i < off.size(); ++i) off[i] += off[i - 1];
        items.resize(pts.size());
        std::vector<int64_t> cur(off.begin(), off.end() - 1);
        for (size_t i = 0; i < pts.size(); ++i) items[cur[cellof[i]]++] = (int32_t)i;
    }
    void coords(const double* p, int64_t* c) const {
        for (int k = 0; k < 3; ++k) {
            const double r = (p[k] - lo[k]) / cell;
            int64_t v = r <= 0 ? 0 : (int64_t)r;
            c[k] = std::min<int64_t>(std::max<int64_t>(v, 0), dims[k] - 1);
        }
    }
    int64_t cell_of(const double* p) const {
        int64_t c[3];
        coords(p, c);
        return (c[2] * dims[1] + c[1]) * dims[0] + c[0];
    }
    int32_t nearest(const double* q) const {
        int64_t qc[3];
        coords(q, qc);
        double bd = INFINITY;
        int32_t bo = INT32_MAX, bf = INT32_MAX;
        const int64_t max_ring = std::max({dims[0], dims[1], dims[2]});
        for (int64_t r = 0; r <= max_ring + 1; ++r) {
            const double ring_min = r > 1 ? (double)(r - 1) * cell : 0.0;
            if (bf != INT32_MAX && ring_min * ring_min > bd) break;
            for (int64_t dz = -r; dz <= r; ++dz)
                for (int64_t dy = -r; dy <= r; ++dy)
                    for (int64_t dx = -r; dx <= r; ++dx) {
                        if (std::max({std::llabs(dx), std::llabs(dy), std::llabs(dz)}) != r) continue;
                        const int64_t cx = qc[0] + dx, cy = qc[1] + dy, cz = qc[2] + dz;
                        if (cx < 0 || cy < 0 || cz < 0 || cx >= dims[0] || cy >= dims[1] || cz >= dims[2]) continue;
                        const int64_t cid = (cz * dims[1] + cy) * dims[0] + cx;
                        for (int64_t i = off[cid]; i < off[cid + 1]; ++i) {
                            const Cand& p = pts[items[i]];
                            const double d[3] = {p.c[0] - q[0], p.c[1] - q[1], p.c[2] - q[2]};
                            const double d2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
                            if (d2 < bd || (d2 == bd && (p.owner < bo || (p.owner == bo && p.facet < bf)))) {
                                bd = d2;
                                bo = p.owner;
                                bf = p.facet;
                            }
                        }
                    }
        }
        return bf;
    }
};
}  // namespace

std::vector<Pair> pair_sister_facets(const MeshData& m) {
    std::vector<Pair> pairs;
    for (int32_t c = 0; c < (int32_t)m.contacts.size() / 2; ++c) {
        const int32_t ta = m.contacts[2 * c], tb = m.contacts[2 * c + 1];
        std::vector<int32_t> sa, sb;
        for (int32_t f = 0; f < m.F; ++f) {
            if (m.facet_tag[f] == ta) sa.push_back(f);
            if (m.facet_tag[f] == tb) sb.push_back(f);
        }
        if (sa.empty() || sb.empty())
            raise(CF_CONFIG, "contact " + m.tags[ta] + "/" + m.tags[tb] + ": side '" + m.tags[sa.empty() ? ta : tb] +
                                 "' has no tagged facets");
        Grid ga, gb;
        auto fill = [&](Grid& g, const std::vector<int32_t>& side) {
            g.pts.resize(side.size());
            for (size_t i = 0; i < side.size(); ++i) {
                const int32_t f = side[i];
                triangle_centroid(m.pos(m.facets[3 * (size_t)f]), m.pos(m.facets[3 * (size_t)f + 1]),
                                  m.pos(m.facets[3 * (size_t)f + 2]), g.pts[i].c);
                g.pts[i].facet = f;
                g.pts[i].owner = m.owner[f];
            }
            g.build();
        };
        fill(ga, sa);
        fill(gb, sb);
        const size_t base = pairs.size();
        pairs.resize(base + sa.size() + sb.size());
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t i = 0; i < (int64_t)sa.size(); ++i) {
            const int32_t nf = gb.nearest(ga.pts[i].c);
            pairs[base + i] = {sa[i], m.owner[nf], c};
        }
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t i = 0; i < (int64_t)sb.size(); ++i) {
            const int32_t nf = ga.nearest(gb.pts[i].c);
            pairs[base + sa.size() + i] = {sb[i], m.owner[nf], c};
        }
    }
    return pairs;
}

// ------------------------------------------------------------------ graph / RCM
Graph build_node_graph(int32_t N, int32_t E, const int32_t* tets) {
    // node -> incident elements, then per node sorted unique neighbours
    std::vector<int64_t> eoff(N + 1, 0);
    for (int64_t i = 0; i < 4 * (int64_t)E; ++i) eoff[tets[i] + 1]++;
    for (int32_t n = 0; n < N; ++n) eoff[n + 1] += eoff[n];
    std::vector<int32_t> einc(4 * (size_t)E);
    {
        std::vector<int64_t> cur(eoff.begin(), eoff.end() - 1);
        for (int64_t i = 0; i < 4 * (int64_t)E; ++i) einc[cur[tets[i]]++] = (int32_t)(i / 4);
    }
    Graph g;
    g.n = N;
    g.off.assign(N + 1, 0);
    // two passes: count, fill
    std::vector<int32_t> deg(N);
#pragma omp parallel
    {
        std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 4096)
        for (int32_t n = 0; n < N; ++n) {
            buf.clear();
            for (int64_t j = eoff[n]; j < eoff[n + 1]; ++j) {
                const int32_t* t = tets + 4 * (size_t)einc[j];
                for (int a = 0; a < 4; ++a)
                    if (t[a] != n) buf.push_back(t[a]);
            }
            std::sort(buf.begin(), buf.end());
            deg[n] = (int32_t)(std::unique(buf.begin(), buf.end()) - buf.begin());
        }
    }
    for (int32_t n = 0; n < N; ++n) g.off[n + 1] = g.off[n] + deg[n];
    g.adj.resize(g.off[N]);
#pragma omp parallel
    {
        std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 4096)
        for (int32_t n = 0; n < N; ++n) {
            buf.clear();
            for (int64_t j = eoff[n]; j < eoff[n + 1]; ++j) {
                const int32_t* t = tets + 4 * (size_t)einc[j];
                for (int a = 0; a < 4; ++a)
                    if (t[a] != n) buf.push_back(t[a]);
            }
            std::sort(buf.begin(), buf.end());
            buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
            std::copy(buf.begin(), buf.end(), g.adj.begin() + g.off[n]);
        }
    }
    return g;
}

namespace {
// The reference's Cuthill-McKee BFS (bfs_levels reorder.hpp:54-88) appends each visited vertex's
// unseen neighbours sorted by (degree, id). Its order within level L+1 is therefore fixed by the
// level-L position of each vertex's first discoverer, then (degree, id) -- the formulation the
// device pass uses (cf_rcm.cu). Here: level sets by BFS, then each level sorted by
// (smallest position among its neighbours in the previous level, degree, id).
struct Levels {
    std::vector<int32_t> dist;  // -1 unvisited in this sweep (only the touched entries are reset)
    std::vector<int32_t> touched;
    explicit Levels(int32_t n) : dist(n, -1) {}
    // BFS from root (set semantics); returns the level sets in discovery-independent order
    int64_t sweep(const Graph& g, int32_t root, std::vector<std::vector<int32_t>>* levels,
                  std::vector<int32_t>* last) {
        for (int32_t v : touched) dist[v] = -1;
        touched.assign(1, root);
        dist[root] = 0;
        std::vector<int32_t> front{root}, next;
        if (levels) levels->assign(1, front);
        int64_t depth = 0;
        for (;;) {
            next.clear();
            for (int32_t v : front)
                for (int64_t j = g.off[v]; j < g.off[v + 1]; ++j) {
                    const int32_t u = g.adj[j];
                    if (dist[u] < 0) {
                        dist[u] = (int32_t)depth + 1;
                        touched.push_back(u);
                        next.push_back(u);
                    }
                }
            if (next.empty()) break;
            ++depth;
            front.swap(next);
            if (levels) levels->push_back(front);
        }
        if (last) *last = front;
        return depth;
    }
};

// pseudo_peripheral reorder.hpp:91-120 (George-Liu): restart from the (degree, id)-smallest vertex
// of the last level while the eccentricity grows
int32_t pseudo_peripheral(const Graph& g, int32_t start, Levels& lv) {
    int32_t node = start;
    int64_t ecc = -1;
    std::vector<int32_t> last;
    for (;;) {
        const int64_t depth = lv.sweep(g, node, nullptr, &last);
        if (depth <= ecc) return node;
        ecc = depth;
        node = *std::min_element(last.begin(), last.end(), [&](int32_t a, int32_t b) {
            return g.degree(a) != g.degree(b) ? g.degree(a) < g.degree(b) : a < b;
        });
    }
}

// Cuthill-McKee order of root's component appended to `order` (positions in `pos`)
void cm_order(const Graph& g, int32_t root, Levels& lv, std::vector<int32_t>& order, std::vector<int64_t>& pos) {
    std::vector<std::vector<int32_t>> levels;
    lv.sweep(g, root, &levels, nullptr);
    pos[root] = (int64_t)order.size();
    order.push_back(root);
    struct Key {
        int64_t parent;
        int32_t deg, id;
    };
    std::vector<Key> keys;
    for (size_t L = 1; L < levels.size(); ++L) {
        keys.clear();
        for (int32_t u : levels[L]) {
            int64_t first = INT64_MAX;  // first discoverer: earliest-placed neighbour one level up
            for (int64_t j = g.off[u]; j < g.off[u + 1]; ++j) {
                const int32_t w = g.adj[j];
                if (lv.dist[w] == (int32_t)L - 1) first = std::min(first, pos[w]);
            }
            keys.push_back({first, g.degree(u), u});
        }
        std::sort(keys.begin(), keys.end(), [](const Key& a, const Key& b) {
            if (a.parent != b.parent) return a.parent < b.parent;
            return a.deg != b.deg ? a.deg < b.deg : a.id < b.id;
        });
        for (const Key& k : keys) {
            pos[k.id] = (int64_t)order.size();
            order.push_back(k.id);
        }
    }
}
}  // namespace

// rcm_permutation reorder.hpp:127-148: components by ascending smallest vertex id, each rooted at
// a pseudo-peripheral vertex (or at the seed when it lies in the component), order reversed
std::vector<int32_t> rcm_permutation(const Graph& g, int32_t seed) {
    const int32_t n = g.n;
    std::vector<int32_t> order;
    order.reserve(n);
    std::vector<int64_t> pos(n, -1);
    Levels lv(n);
    for (int32_t v = 0; v < n; ++v) {
        if (pos[v] >= 0) continue;
        int32_t root;
        if (seed >= 0 && seed < n && pos[seed] < 0) {
            lv.sweep(g, v, nullptr, nullptr);
            root = lv.dist[seed] >= 0 ? seed : pseudo_peripheral(g, v, lv);
        } else {
            root = pseudo_peripheral(g, v, lv);
        }
        cm_order(g, root, lv, order, pos);
    }
    std::vector<int32_t> new_of_old(n);
    for (int32_t i = 0; i < n; ++i) new_of_old[order[i]] = n - 1 - i;
    return new_of_old;
}

int64_t bandwidth(const Graph& g, const int32_t* p) {
    int64_t bw = 0;
    for (int32_t u = 0; u < g.n; ++u)
        for (int64_t j = g.off[u]; j < g.off[u + 1]; ++j) {
            const int32_t v = g.adj[j];
            const int64_t a = p ? p[u] : u, b = p ? p[v] : v;
            bw = std::max<int64_t>(bw, (int64_t)std::llabs(a - b));
        }
    return bw;
}

// ------------------------------------------------------------------ RCB
std::vector<int32_t> partition_rcb(const MeshData& m, int32_t parts) {
    if (parts < 1) raise(CF_INVALID_ARG, "parts must be >= 1");
    const int64_t E = m.E;
    // contiguous (centroid, id) records: the bisections stream them instead of
    // chasing ids; (coordinate, id) is a total order, so each split takes the
    // same set of elements whatever the record order
    struct Rec {
        double c[3];
        int32_t id;
    };
    std::vector<Rec, UninitAlloc<Rec>> rec(E);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        const int32_t* t = &m.tets[4 * (size_t)e];
        for (int k = 0; k < 3; ++k)
            rec[e].c[k] = (((m.pos(t[0])[k] + m.pos(t[1])[k]) + m.pos(t[2])[k]) + m.pos(t[3])[k]) * 0.25;
        rec[e].id = (int32_t)e;
    }
    std::vector<int32_t> part(E, 0);
    struct Job {
        int64_t lo, hi;
        int32_t first, count;
    };
    std::vector<Job> stack{{0, E, 0, parts}};
    while (!stack.empty()) {
        Job j = stack.back();
        stack.pop_back();
        if (j.count == 1) {
#pragma omp parallel for schedule(static)
            for (int64_t i = j.lo; i < j.hi; ++i) part[rec[i].id] = j.first;
            continue;
        }
        double lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY;
#pragma omp parallel for schedule(static) reduction(min : lo0, lo1, lo2) reduction(max : hi0, hi1, hi2)
        for (int64_t i = j.lo; i < j.hi; ++i) {
            lo0 = std::min(lo0, rec[i].c[0]);
            lo1 = std::min(lo1, rec[i].c[1]);
            lo2 = std::min(lo2, rec[i].c[2]);
            hi0 = std::max(hi0, rec[i].c[0]);
            hi1 = std::max(hi1, rec[i].c[1]);
            hi2 = std::max(hi2, rec[i].c[2]);
        }
        const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
        int axis = 0;
        for (int k = 1; k < 3; ++k)
            if (hi[k] - lo[k] > hi[axis] - lo[axis]) axis = k;
        const int32_t left = j.count / 2;
        const int64_t n = j.hi - j.lo;
        const int64_t nl = n * left / j.count;
        auto cmp = [axis](const Rec& a, const Rec& b) {
            return a.c[axis] != b.c[axis] ? a.c[axis] < b.c[axis] : a.id < b.id;
        };
        __gnu_parallel::nth_element(rec.begin() + j.lo, rec.begin() + j.lo + nl, rec.begin() + j.hi, cmp);
        stack.push_back({j.lo + nl, j.hi, j.first + left, j.count - left});
        stack.push_back({j.lo, j.lo + nl, j.first, left});
    }
    return part;
}

// ------------------------------------------------------------------ fixtures
static inline uint64_t splitmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
double counter_uniform(uint64_t seed, uint64_t key) {
    const uint64_t z = splitmix(seed * 0x9E3779B97F4A7C15ull + splitmix(key + 0x632BE59BD9B4E019ull));
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

void generate_fixture(int kind, int n, double radius, double jitter, uint64_t seed, uint64_t perm_seed,
                      cf_fixture* out) {
    if (n < 1 || n > 1024) raise(CF_INVALID_ARG, "fixture n out of range [1, 1024]");
    if (kind != 0 && kind != 1) raise(CF_INVALID_ARG, "fixture kind must be 0 (cube) or 1 (casting)");
    const int64_t P = n + 1;
    const double h = 1.0 / n;
    // cell region: casting iff sum (2i+1-n)^2 <= 4 r^2 n^2 (cell-centre test); exact in
    // integers when 100 r^2 is an integer (r = 0.35 -> 49)
    const int64_t r100 = (int64_t)std::llround(radius * radius * 100.0);
    const bool exact = std::fabs(radius * radius * 100.0 - (double)r100) < 1e-9;
    auto cell_region = [&](int64_t i, int64_t j, int64_t k) -> int32_t {
        if (kind == 0) return 0;
        const int64_t a = 2 * i + 1 - n, b = 2 * j + 1 - n, c = 2 * k + 1 - n;
        const int64_t s = a * a + b * b + c * c;
        const bool cast = exact ? (100 * s <= 4 * r100 * (int64_t)n * n)
                                : ((double)s <= 4.0 * radius * radius * (double)n * n);
        return cast ? 0 : 1;  // region 0 = casting, 1 = mould
    };
    const int64_t C = (int64_t)n * n * n;
    std::vector<uint8_t> creg(C);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) creg[c] = (uint8_t)cell_region(c % n, (c / n) % n, c / ((int64_t)n * n));
    auto cidx = [&](int64_t i, int64_t j, int64_t k) { return i + n * (j + (int64_t)n * k); };
    // node copies per grid point: bit r set if region r touches the point
    const int64_t G = P * P * P;
    std::vector<uint8_t> touch(G, 0);
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const uint8_t bit = (uint8_t)(1u << creg[cidx(i, j, k)]);
                for (int d = 0; d < 8; ++d)
                    touch[(i + (d & 1)) + P * ((j + ((d >> 1) & 1)) + P * (k + ((d >> 2) & 1)))] |= bit;
            }
    std::vector<int64_t> first(G + 1, 0);
    for (int64_t g = 0; g < G; ++g) first[g + 1] = first[g] + __builtin_popcount(touch[g]);
    const int64_t N = first[G];
    auto node_id = [&](int64_t g, int32_t reg) -> int64_t {
        // copies ordered by region id
        return first[g] + (reg == 1 && (touch[g] & 1) ? 1 : 0);
    };
    // Kuhn split: 6 tets per cell along the axis permutations (a,b,c)
    static const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int64_t E = 6 * C;
    // facets: count first
    auto nb_region = [&](int64_t i, int64_t j, int64_t k) -> int32_t {  // -1 outside
        if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n) return -1;
        return creg[cidx(i, j, k)];
    };
    std::vector<int64_t> fcount(C + 1, 0);
    for (int64_t c = 0; c < C; ++c) {
        const int64_t i = c % n, j = (c / n) % n, k = c / ((int64_t)n * n);
        const int32_t rg = creg[c];
        int cnt = 0;
        for (int t = 0; t < 6; ++t) {
            const int a = perm[t][0], cc = perm[t][2];
            int64_t lo[3] = {i, j, k}, hi[3] = {i, j, k};
            lo[cc] -= 1;
            hi[a] += 1;
            const int32_t r1 = nb_region(lo[0], lo[1], lo[2]), r2 = nb_region(hi[0], hi[1], hi[2]);
            if (r1 != rg) ++cnt;
            if (r2 != rg) ++cnt;
        }
        fcount[c + 1] = fcount[c] + cnt;
    }
    const int64_t F = fcount[C];
    if (N > INT32_MAX || E > INT32_MAX || F > INT32_MAX) raise(CF_INVALID_ARG, "fixture too large for int32 ids");
    out->n_nodes = (int32_t)N;
    out->n_elems = (int32_t)E;
    out->n_facets = (int32_t)F;
    if (!out->coords || !out->tets || !out->region || !out->facets || !out->facet_tag) return;  // size query

    // node permutation
    std::vector<int32_t> nperm, eperm;
    if (perm_seed) {
        nperm.resize(N);
        std::iota(nperm.begin(), nperm.end(), 0);
        uint64_t s = perm_seed;
        for (int64_t i = N - 1; i > 0; --i) {
            s = splitmix(s + 0x9E3779B97F4A7C15ull);
            std::swap(nperm[i], nperm[s % (uint64_t)(i + 1)]);
        }
        eperm.resize(E);
        std::iota(eperm.begin(), eperm.end(), 0);
        s = splitmix(perm_seed ^ 0xD1B54A32D192ED03ull);
        for (int64_t i = E - 1; i > 0; --i) {
            s = splitmix(s + 0x9E3779B97F4A7C15ull);
            std::swap(eperm[i], eperm[s % (uint64_t)(i + 1)]);
        }
    }
    auto NID = [&](int64_t id) -> int32_t { return perm_seed ? nperm[id] : (int32_t)id; };

#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < G; ++g) {
        const int64_t i = g % P, j = (g / P) % P, k = g / (P * P);
        double x[3] = {i * h, j * h, k * h};
        const int64_t gi[3] = {i, j, k};
        if (jitter != 0 && i > 0 && j > 0 && k > 0 && i < n && j < n && k < n)
            for (int d = 0; d < 3; ++d)
                x[d] = (double)gi[d] * h + (2.0 * counter_uniform(seed, 3 * (uint64_t)g + d) - 1.0) * jitter * h;
        for (int64_t id = first[g]; id < first[g + 1]; ++id) {
            const int32_t nid = NID(id);
            for (int d = 0; d < 3; ++d) out->coords[3 * (size_t)nid + d] = x[d];
            if (out->node_grid) out->node_grid[nid] = (int32_t)g;
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        const int64_t i = c % n, j = (c / n) % n, k = c / ((int64_t)n * n);
        const int32_t rg = creg[c];
        for (int t = 0; t < 6; ++t) {
            const int a = perm[t][0], b = perm[t][1];
            int64_t v[4][3] = {{i, j, k}, {i, j, k}, {i, j, k}, {i + 1, j + 1, k + 1}};
            v[1][a] += 1;
            v[2][a] += 1;
            v[2][b] += 1;
            const int64_t e = 6 * c + t;
            const int64_t eo = perm_seed ? eperm[e] : e;
            for (int q = 0; q < 4; ++q)
                out->tets[4 * (size_t)eo + q] = NID(node_id(v[q][0] + P * (v[q][1] + P * v[q][2]), rg));
            out->region[eo] = rg;
        }
        int64_t fi = fcount[c];
        for (int t = 0; t < 6; ++t) {
            const int a = perm[t][0], b = perm[t][1], cc = perm[t][2];
            int64_t v[4][3] = {{i, j, k}, {i, j, k}, {i, j, k}, {i + 1, j + 1, k + 1}};
            v[1][a] += 1;
            v[2][a] += 1;
            v[2][b] += 1;
            int64_t lo[3] = {i, j, k}, hi[3] = {i, j, k};
            lo[cc] -= 1;
            hi[a] += 1;
            const int32_t r1 = nb_region(lo[0], lo[1], lo[2]), r2 = nb_region(hi[0], hi[1], hi[2]);
            const int faces[2][3] = {{0, 1, 2}, {1, 2, 3}};
            const int32_t nr[2] = {r1, r2};
            for (int s = 0; s < 2; ++s) {
                if (nr[s] == rg) continue;
                for (int q = 0; q < 3; ++q) {
                    const int64_t* p = v[faces[s][q]];
                    out->facets[3 * (size_t)fi + q] = NID(node_id(p[0] + P * (p[1] + P * p[2]), rg));
                }
                out->facet_tag[fi] = nr[s] < 0 ? 0 : (rg == 0 ? 1 : 2);
                ++fi;
            }
        }
    }
}

}  // namespace cfb
