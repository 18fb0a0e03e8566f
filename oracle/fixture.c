/* fixture.c — TEST INFRASTRUCTURE: the synthetic BASELINE workloads restated for the CPU
 * checkers, so the reference arm of bench.py and its CPU baseline never load the product
 * library (libcastfem_b200.so). Built into oracle/liboracle.so (pinned against the product's
 * cf_generate_fixture bit for bit by tests/test_oracle_pin.py) and into the reference
 * benchmark binary oracle/_ref/ref_bench.
 *
 * The rules are SURVEY §8(d)'s generator rules (the reference ships no fixtures: its bench
 * module exists only as specification, "cube(n=1) -> 6-tet cube, 8 nodes
 * [Kuhn subdivision]", "6·n³"):
 *   - structured unit cube of n^3 cells, grid point (i,j,k) at (i,j,k)/n, each cell split into
 *     the 6 Kuhn tets {v000, v000+e_a, v000+e_a+e_b, v111} over the axis permutations (a,b,c);
 *   - casting: a cell is cast (region 0) iff its centre lies within `radius` of the box centre,
 *     tested exactly in integers as sum (2i+1-n)^2 <= 4 r^2 n^2 when 100 r^2 is an integer,
 *     else mould (region 1); a grid point touched by both regions carries one node per region
 *     (regions are node-disjoint, mesh.hpp:129-144), copies ordered by region id;
 *   - boundary facets are the tet faces on a cell face whose neighbour is outside the box
 *     (tag 0 "outer") or of the other region (tag 1 "cast_if" on the cast side, 2 "mold_if" on
 *     the mould side), in (cell, tet, face) order;
 *   - jitter: interior grid points move by U(-jitter h, +jitter h) per coordinate, keyed by
 *     (seed, 3 g + d) with g the grid point index, so both copies of a node move together;
 *   - perm_seed != 0: seeded Fisher-Yates permutations of the node and element numbering.
 *
 * Window (bench sample of a mesh too large for the reference's host memory): only the cells
 * [i0,i1) x [j0,j1) x [k0,k1) of the n^3 grid are generated, with the full mesh's h, regions,
 * jitter and noise keys (node_grid holds the GLOBAL grid point index); faces toward cells
 * outside the window but inside the box get no facet (adiabatic cut planes). The full window
 * is the full mesh, numbering included.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/castfem_b200.h"

static uint64_t fx_splitmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* uniform [0,1) keyed by (seed, key): counter-based, independent of numbering */
double or_counter_uniform(uint64_t seed, uint64_t key) {
    const uint64_t z = fx_splitmix(seed * 0x9E3779B97F4A7C15ull + fx_splitmix(key + 0x632BE59BD9B4E019ull));
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

void or_counter_uniform_array(uint64_t seed, const int64_t* keys, int64_t n, double lo, double hi, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * or_counter_uniform(seed, (uint64_t)keys[i]);
}

static const int kPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

typedef struct {
    int kind, n;
    int64_t i0, j0, k0, wx, wy, wz;  /* window origin and size in cells */
    int64_t r100;
    int exact;
    double radius;
} FxGrid;

static int32_t fx_cell_region(const FxGrid* g, int64_t i, int64_t j, int64_t k) {
    if (g->kind == 0) return 0;
    const int64_t n = g->n;
    const int64_t a = 2 * i + 1 - n, b = 2 * j + 1 - n, c = 2 * k + 1 - n;
    const int64_t s = a * a + b * b + c * c;
    const int cast = g->exact ? (100 * s <= 4 * g->r100 * n * n)
                              : ((double)s <= 4.0 * g->radius * g->radius * (double)n * (double)n);
    return cast ? 0 : 1;
}

/* region of the neighbour cell (global indices): -1 outside the box, -2 outside the window */
static int32_t fx_nb_region(const FxGrid* g, int64_t i, int64_t j, int64_t k) {
    if (i < 0 || j < 0 || k < 0 || i >= g->n || j >= g->n || k >= g->n) return -1;
    if (i < g->i0 || j < g->j0 || k < g->k0 || i >= g->i0 + g->wx || j >= g->j0 + g->wy || k >= g->k0 + g->wz)
        return -2;
    return fx_cell_region(g, i, j, k);
}

int or_generate_fixture(int32_t kind, int32_t n, double radius, double jitter, uint64_t seed, uint64_t perm_seed,
                        const int32_t* window, cf_fixture* out) {
    if (n < 1 || n > 1024 || (kind != 0 && kind != 1) || !out) return CF_INVALID_ARG;
    FxGrid g;
    g.kind = kind;
    g.n = n;
    g.radius = radius;
    g.r100 = llround(radius * radius * 100.0);
    g.exact = fabs(radius * radius * 100.0 - (double)g.r100) < 1e-9;
    if (window) {
        g.i0 = window[0], g.wx = window[1] - window[0];
        g.j0 = window[2], g.wy = window[3] - window[2];
        g.k0 = window[4], g.wz = window[5] - window[4];
        if (g.i0 < 0 || g.j0 < 0 || g.k0 < 0 || g.wx < 1 || g.wy < 1 || g.wz < 1 || g.i0 + g.wx > n ||
            g.j0 + g.wy > n || g.k0 + g.wz > n)
            return CF_INVALID_ARG;
    } else {
        g.i0 = g.j0 = g.k0 = 0;
        g.wx = g.wy = g.wz = n;
    }
    const double h = 1.0 / n;
    const int64_t PG = (int64_t)n + 1;                                  /* global grid points per axis */
    const int64_t PX = g.wx + 1, PY = g.wy + 1, PZ = g.wz + 1;          /* window grid points */
    const int64_t C = g.wx * g.wy * g.wz, G = PX * PY * PZ;
    uint8_t* creg = (uint8_t*)malloc((size_t)C);
    uint8_t* touch = (uint8_t*)calloc((size_t)G, 1);
    int64_t* first = (int64_t*)malloc(sizeof(int64_t) * (size_t)(G + 1));
    int64_t* fcount = (int64_t*)malloc(sizeof(int64_t) * (size_t)(C + 1));
    if (!creg || !touch || !first || !fcount) {
        free(creg), free(touch), free(first), free(fcount);
        return CF_INVALID_ARG;
    }
#define CIDX(li, lj, lk) ((li) + g.wx * ((lj) + g.wy * (lk)))
#define GIDX(li, lj, lk) ((li) + PX * ((lj) + PY * (lk)))
    for (int64_t c = 0; c < C; ++c)
        creg[c] = (uint8_t)fx_cell_region(&g, g.i0 + c % g.wx, g.j0 + (c / g.wx) % g.wy, g.k0 + c / (g.wx * g.wy));
    for (int64_t lk = 0; lk < g.wz; ++lk)
        for (int64_t lj = 0; lj < g.wy; ++lj)
            for (int64_t li = 0; li < g.wx; ++li) {
                const uint8_t bit = (uint8_t)(1u << creg[CIDX(li, lj, lk)]);
                for (int d = 0; d < 8; ++d) touch[GIDX(li + (d & 1), lj + ((d >> 1) & 1), lk + ((d >> 2) & 1))] |= bit;
            }
    first[0] = 0;
    for (int64_t q = 0; q < G; ++q) first[q + 1] = first[q] + __builtin_popcount(touch[q]);
    const int64_t N = first[G];
    fcount[0] = 0;
    for (int64_t c = 0; c < C; ++c) {
        const int64_t i = g.i0 + c % g.wx, j = g.j0 + (c / g.wx) % g.wy, k = g.k0 + c / (g.wx * g.wy);
        const int32_t rg = creg[c];
        int cnt = 0;
        for (int t = 0; t < 6; ++t) {
            const int a = kPerm[t][0], cc = kPerm[t][2];
            int64_t lo[3] = {i, j, k}, hi[3] = {i, j, k};
            lo[cc] -= 1;
            hi[a] += 1;
            const int32_t r1 = fx_nb_region(&g, lo[0], lo[1], lo[2]), r2 = fx_nb_region(&g, hi[0], hi[1], hi[2]);
            cnt += (r1 != rg && r1 != -2) + (r2 != rg && r2 != -2);
        }
        fcount[c + 1] = fcount[c] + cnt;
    }
    const int64_t E = 6 * C, F = fcount[C];
    if (N > INT32_MAX || E > INT32_MAX || F > INT32_MAX) {
        free(creg), free(touch), free(first), free(fcount);
        return CF_INVALID_ARG;
    }
    out->n_nodes = (int32_t)N;
    out->n_elems = (int32_t)E;
    out->n_facets = (int32_t)F;
    if (!out->coords || !out->tets || !out->region || !out->facets || !out->facet_tag) { /* size query */
        free(creg), free(touch), free(first), free(fcount);
        return CF_OK;
    }
    int32_t* nperm = NULL;
    int32_t* eperm = NULL;
    if (perm_seed) {
        nperm = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N ? N : 1));
        eperm = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
        for (int64_t q = 0; q < N; ++q) nperm[q] = (int32_t)q;
        uint64_t s = perm_seed;
        for (int64_t q = N - 1; q > 0; --q) {
            s = fx_splitmix(s + 0x9E3779B97F4A7C15ull);
            const int64_t r = (int64_t)(s % (uint64_t)(q + 1));
            const int32_t tmp = nperm[q];
            nperm[q] = nperm[r];
            nperm[r] = tmp;
        }
        for (int64_t q = 0; q < E; ++q) eperm[q] = (int32_t)q;
        s = fx_splitmix(perm_seed ^ 0xD1B54A32D192ED03ull);
        for (int64_t q = E - 1; q > 0; --q) {
            s = fx_splitmix(s + 0x9E3779B97F4A7C15ull);
            const int64_t r = (int64_t)(s % (uint64_t)(q + 1));
            const int32_t tmp = eperm[q];
            eperm[q] = eperm[r];
            eperm[r] = tmp;
        }
    }
#define NID(id) (nperm ? nperm[(id)] : (int32_t)(id))
    /* a region's copy of window grid point q: copies ordered by region id */
#define NODE(q, reg) (first[(q)] + (((reg) == 1 && (touch[(q)] & 1)) ? 1 : 0))
    for (int64_t q = 0; q < G; ++q) {
        const int64_t li = q % PX, lj = (q / PX) % PY, lk = q / (PX * PY);
        const int64_t gi[3] = {g.i0 + li, g.j0 + lj, g.k0 + lk};
        const int64_t gg = gi[0] + PG * (gi[1] + PG * gi[2]);
        double x[3] = {gi[0] * h, gi[1] * h, gi[2] * h};
        if (jitter != 0 && gi[0] > 0 && gi[1] > 0 && gi[2] > 0 && gi[0] < n && gi[1] < n && gi[2] < n)
            for (int d = 0; d < 3; ++d)
                x[d] = (double)gi[d] * h + (2.0 * or_counter_uniform(seed, 3 * (uint64_t)gg + d) - 1.0) * jitter * h;
        for (int64_t id = first[q]; id < first[q + 1]; ++id) {
            const int32_t nid = NID(id);
            for (int d = 0; d < 3; ++d) out->coords[3 * (size_t)nid + d] = x[d];
            if (out->node_grid) out->node_grid[nid] = (int32_t)gg;
        }
    }
    for (int64_t c = 0; c < C; ++c) {
        const int64_t li = c % g.wx, lj = (c / g.wx) % g.wy, lk = c / (g.wx * g.wy);
        const int64_t i = g.i0 + li, j = g.j0 + lj, k = g.k0 + lk;
        const int32_t rg = creg[c];
        int64_t fi = fcount[c];
        for (int t = 0; t < 6; ++t) {
            const int a = kPerm[t][0], b = kPerm[t][1];
            int64_t v[4][3] = {{li, lj, lk}, {li, lj, lk}, {li, lj, lk}, {li + 1, lj + 1, lk + 1}};
            v[1][a] += 1;
            v[2][a] += 1;
            v[2][b] += 1;
            const int64_t e = 6 * c + t;
            const int64_t eo = eperm ? eperm[e] : e;
            for (int q = 0; q < 4; ++q) out->tets[4 * (size_t)eo + q] = NID(NODE(GIDX(v[q][0], v[q][1], v[q][2]), rg));
            out->region[eo] = rg;
        }
        for (int t = 0; t < 6; ++t) {
            const int a = kPerm[t][0], b = kPerm[t][1], cc = kPerm[t][2];
            int64_t v[4][3] = {{li, lj, lk}, {li, lj, lk}, {li, lj, lk}, {li + 1, lj + 1, lk + 1}};
            v[1][a] += 1;
            v[2][a] += 1;
            v[2][b] += 1;
            int64_t lo[3] = {i, j, k}, hi[3] = {i, j, k};
            lo[cc] -= 1;
            hi[a] += 1;
            const int32_t nr[2] = {fx_nb_region(&g, lo[0], lo[1], lo[2]), fx_nb_region(&g, hi[0], hi[1], hi[2])};
            static const int faces[2][3] = {{0, 1, 2}, {1, 2, 3}};
            for (int s = 0; s < 2; ++s) {
                if (nr[s] == rg || nr[s] == -2) continue;
                for (int q = 0; q < 3; ++q) {
                    const int64_t* p = v[faces[s][q]];
                    out->facets[3 * (size_t)fi + q] = NID(NODE(GIDX(p[0], p[1], p[2]), rg));
                }
                out->facet_tag[fi] = nr[s] < 0 ? 0 : (rg == 0 ? 1 : 2);
                ++fi;
            }
        }
    }
#undef NID
#undef NODE
#undef CIDX
#undef GIDX
    free(nperm), free(eperm), free(creg), free(touch), free(first), free(fcount);
    return CF_OK;
}
