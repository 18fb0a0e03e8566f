/*
 * castfem_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference castfem explicit step
 * (arXiv 1005.3158; /root/reference/proj/include/castfem/, cited below
 * relative to that directory). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's
 * library; the product path never calls it.
 *
 * Parity is PINNED: tests/test_oracle_pin.py runs this restatement and the
 * reference itself (oracle/_ref/castfem_ref, built from the reference headers
 * by oracle/Makefile) on the same seeded meshes and requires bitwise-equal
 * nodal temperatures; tests/golden/ holds vectors produced by the reference.
 *
 * Build with -ffp-contract=off (no FMA), matching the reference's CMake
 * Release build (no -march), which is bitwise stable (SURVEY §0 trap 10).
 *
 * Semantics restated:
 *   geometry      tet_geometry            geometry.hpp:48-77
 *   tables        PiecewiseLinear         material.hpp:21-47
 *   enthalpy      MaterialTable::enthalpy material.hpp:89-102, finalize :104-119
 *   Lemmon        apparent_heat_capacity  fem.hpp:26-45
 *   element       element_accumulate      fem.hpp:57-70
 *   facet         facet_flux_accumulate   fem.hpp:74-79, interface blocked.hpp:485-490
 *   blocks        build_worker_model      blocked.hpp:156-361 (slots, merge CSR)
 *   assemble      assemble_blocks         blocked.hpp:454-498
 *   merge         merge_blocks            blocked.hpp:502-515
 *   ambient       refresh_ambient         blocked.hpp:441-449 (one-step lag)
 *   update        update_fields           blocked.hpp:519-538, explicit_update fem.hpp:107-114
 *   step          blocked_step            blocked.hpp:542-550
 *   driver        solve_serial            blocked.hpp:650-696
 *   mesh checks   finalize_mesh           mesh.hpp:148-207, node_regions :129-144
 *   sisters       pair_sister_facets      mesh.hpp:456-478 (exact nearest, same ties)
 *   workers       parallel_solve: per-node sum over parts in
 *                 ascending part id of the part's merged partial.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/castfem_b200.h"

#define OR_EXPORT __attribute__((visibility("default")))

int cmpi(const void* x, const void* y);

static char g_err[512];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
OR_EXPORT const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ vec3 */
typedef struct { double x, y, z; } v3;
static v3 vsub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 vadd(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 vmul(v3 a, double s) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 vcross(v3 a, v3 b) {
    v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
    return r;
}
static double vnorm(v3 a) { return sqrt(vdot(a, a)); }
static v3 node_pos(const cf_mesh_desc* m, int n) {
    v3 r = {m->coords[3 * (size_t)n], m->coords[3 * (size_t)n + 1], m->coords[3 * (size_t)n + 2]};
    return r;
}

/* tet_geometry geometry.hpp:48-77 */
typedef struct { double vol; v3 g[4]; double min_edge, max_edge; } geom_t;
static int tet_geom(v3 p0, v3 p1, v3 p2, v3 p3, geom_t* g) {
    v3 e1 = vsub(p1, p0), e2 = vsub(p2, p0), e3 = vsub(p3, p0);
    double det = vdot(e1, vcross(e2, e3));
    g->vol = det / 6.0;
    v3 p[4] = {p0, p1, p2, p3};
    g->min_edge = g->max_edge = vnorm(vsub(p1, p0));
    for (int a = 0; a < 4; ++a)
        for (int b = a + 1; b < 4; ++b) {
            double len = vnorm(vsub(p[b], p[a]));
            if (len < g->min_edge) g->min_edge = len;
            if (len > g->max_edge) g->max_edge = len;
        }
    double eps = 1e-12 * g->max_edge * g->max_edge * g->max_edge;
    if (!(g->vol > eps)) return CF_DEGENERATE;
    g->g[1] = vmul(vcross(e2, e3), 1.0 / det);
    g->g[2] = vmul(vcross(e3, e1), 1.0 / det);
    g->g[3] = vmul(vcross(e1, e2), 1.0 / det);
    g->g[0] = vmul(vadd(vadd(g->g[1], g->g[2]), g->g[3]), -1.0);
    return CF_OK;
}

/* ------------------------------------------------------------ tables */
/* PiecewiseLinear::operator() material.hpp:30-38 */
static double pl_eval(const cf_table* t, double x) {
    if (t->n <= 1) return t->y[0];
    if (x <= t->x[0]) return t->y[0];
    if (x >= t->x[t->n - 1]) return t->y[t->n - 1];
    int i = 0; /* upper_bound - 1 */
    while (i + 1 < t->n && t->x[i + 1] <= x) ++i;
    double f = (x - t->x[i]) / (t->x[i + 1] - t->x[i]);
    return t->y[i] + f * (t->y[i + 1] - t->y[i]);
}

typedef struct {
    const cf_material* m;
    double ref;       /* enthalpy_ref_ */
    double* cum;      /* cumulative_ */
    double range_lo, range_hi;
} mat_t;

static int table_ok(const cf_table* t) {
    if (t->n < 1 || !t->x || !t->y) return 0;
    for (int i = 1; i < t->n; ++i)
        if (!(t->x[i] > t->x[i - 1])) return 0;
    return 1;
}

/* MaterialTable::finalize material.hpp:104-119 (+ range_min/max :75-86) */
static int mat_init(const cf_material* m, mat_t* o) {
    o->m = m;
    if (!table_ok(&m->c) || !table_ok(&m->k)) return fail(CF_CONFIG, "empty or inconsistent table");
    if (!(m->rho > 0)) return fail(CF_CONFIG, "rho must be positive");
    for (int i = 0; i < m->c.n; ++i)
        if (m->c.y[i] <= 0) return fail(CF_CONFIG, "c(T) must be positive");
    for (int i = 0; i < m->k.n; ++i)
        if (m->k.y[i] <= 0) return fail(CF_CONFIG, "k(T) must be positive");
    if (m->latent_heat < 0) return fail(CF_CONFIG, "latent_heat must be non-negative");
    if (m->latent_heat > 0 && !(m->solidus < m->liquidus))
        return fail(CF_CONFIG, "phase change requires solidus < liquidus");
    o->ref = m->c.n <= 1 ? 0.0 : m->c.x[0];
    int nc = m->c.n > 1 ? m->c.n : 1;
    o->cum = (double*)calloc(nc, sizeof(double));
    for (int i = 1; i < m->c.n; ++i)
        o->cum[i] = o->cum[i - 1] + 0.5 * (m->c.y[i] + m->c.y[i - 1]) * (m->c.x[i] - m->c.x[i - 1]);
    o->range_lo = -INFINITY;
    o->range_hi = INFINITY;
    if (m->c.n > 1) { if (m->c.x[0] > o->range_lo) o->range_lo = m->c.x[0]; }
    if (m->k.n > 1) { if (m->k.x[0] > o->range_lo) o->range_lo = m->k.x[0]; }
    if (m->c.n > 1) { if (m->c.x[m->c.n - 1] < o->range_hi) o->range_hi = m->c.x[m->c.n - 1]; }
    if (m->k.n > 1) { if (m->k.x[m->k.n - 1] < o->range_hi) o->range_hi = m->k.x[m->k.n - 1]; }
    return CF_OK;
}

/* melt_fraction material.hpp:69-72 ; std::clamp(v, lo, hi) */
static double melt_fraction(const cf_material* m, double T) {
    if (!(m->latent_heat > 0)) return 0;
    double v = (T - m->solidus) / (m->liquidus - m->solidus);
    return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
}

/* enthalpy material.hpp:89-102 */
static double enthalpy(const mat_t* mt, double T) {
    const cf_material* m = mt->m;
    double sensible;
    if (m->c.n <= 1) {
        sensible = m->c.y[0] * (T - mt->ref);
    } else {
        const double* xs = m->c.x;
        int n = m->c.n;
        double Tc = T < xs[0] ? xs[0] : (xs[n - 1] < T ? xs[n - 1] : T);
        int ub = 0; /* upper_bound index */
        while (ub < n && xs[ub] <= Tc) ++ub;
        int i = (ub < n - 1 ? ub : n - 1) - 1;
        sensible = mt->cum[i] + 0.5 * (m->c.y[i] + pl_eval(&m->c, Tc)) * (Tc - xs[i]);
    }
    return sensible + m->latent_heat * melt_fraction(m, T);
}

/* apparent_heat_capacity fem.hpp:26-45 */
static double apparent_c(const geom_t* g, const double* Tn, const double* Hn, const cf_material* m) {
    int lo = 0, hi = 0;
    for (int a = 1; a < 4; ++a) {
        if (Tn[a] < Tn[lo]) lo = a;
        if (Tn[a] > Tn[hi]) hi = a;
    }
    double range = Tn[hi] - Tn[lo];
    if (range <= 0) return pl_eval(&m->c, 0.25 * (Tn[0] + Tn[1] + Tn[2] + Tn[3]));
    v3 gt = {0, 0, 0}, gh = {0, 0, 0};
    for (int a = 0; a < 4; ++a) {
        gt = vadd(gt, vmul(g->g[a], Tn[a]));
        gh = vadd(gh, vmul(g->g[a], Hn[a]));
    }
    double gt2 = vdot(gt, gt);
    double scale = range / g->max_edge;
    if (gt2 < 1e-14 * scale * scale) return (Hn[hi] - Hn[lo]) / range;
    return sqrt(vdot(gh, gh) / gt2);
}

/* ------------------------------------------------------------ mesh prep */
typedef struct { int32_t k[3]; int32_t facet; int32_t owner; int32_t count; } fslot;
static uint64_t key_hash(const int32_t* k) {
    uint64_t h = (uint64_t)(uint32_t)k[0] * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)(uint32_t)k[1] + 0x7F4A7C159E3779B9ull + (h << 6) + (h >> 2);
    h ^= (uint64_t)(uint32_t)k[2] * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
    return h;
}
static void sort3(int32_t* k) {
    int32_t t;
    if (k[0] > k[1]) { t = k[0]; k[0] = k[1]; k[1] = t; }
    if (k[1] > k[2]) { t = k[1]; k[1] = k[2]; k[2] = t; }
    if (k[0] > k[1]) { t = k[0]; k[0] = k[1]; k[1] = t; }
}

typedef struct {
    int N, E, F;
    int32_t* tets;      /* oriented */
    int32_t* owner;     /* facet owner */
    int32_t* node_region;
    geom_t* geom;
} prep_t;

/* finalize_mesh mesh.hpp:148-207 (orientation swap, degeneracy, regions, owners) */
static int prep_mesh(const cf_mesh_desc* m, int n_materials, prep_t* p) {
    p->N = m->n_nodes; p->E = m->n_elems; p->F = m->n_facets;
    for (int64_t i = 0; i < 3 * (int64_t)p->N; ++i)
        if (!isfinite(m->coords[i])) return fail(CF_VALIDATION, "non-finite node coordinate");
    p->tets = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(p->E > 0 ? p->E : 1));
    p->geom = (geom_t*)malloc(sizeof(geom_t) * (size_t)(p->E > 0 ? p->E : 1));
    p->owner = (int32_t*)malloc(sizeof(int32_t) * (size_t)(p->F > 0 ? p->F : 1));
    p->node_region = (int32_t*)malloc(sizeof(int32_t) * (size_t)(p->N > 0 ? p->N : 1));
    for (int e = 0; e < p->E; ++e) {
        int32_t* t = p->tets + 4 * (size_t)e;
        for (int a = 0; a < 4; ++a) {
            t[a] = m->tets[4 * (size_t)e + a];
            if (t[a] < 0 || t[a] >= p->N) return fail(CF_VALIDATION, "element references node outside range");
        }
        for (int a = 0; a < 4; ++a)
            for (int b = a + 1; b < 4; ++b)
                if (t[a] == t[b]) return fail(CF_VALIDATION, "element has repeated node");
        if (m->region[e] < 0) return fail(CF_VALIDATION, "negative region id");
        v3 p0 = node_pos(m, t[0]), p1 = node_pos(m, t[1]), p2 = node_pos(m, t[2]), p3 = node_pos(m, t[3]);
        double sv = vdot(vsub(p1, p0), vcross(vsub(p2, p0), vsub(p3, p0))) / 6.0;
        if (sv < 0) { int32_t s = t[2]; t[2] = t[3]; t[3] = s; }
        if (tet_geom(node_pos(m, t[0]), node_pos(m, t[1]), node_pos(m, t[2]), node_pos(m, t[3]),
                     &p->geom[e]) != CF_OK)
            return fail(CF_DEGENERATE, "degenerate tetrahedron");
    }
    for (int n = 0; n < p->N; ++n) p->node_region[n] = -1;
    for (int e = 0; e < p->E; ++e)
        for (int a = 0; a < 4; ++a) {
            int n = p->tets[4 * (size_t)e + a];
            if (p->node_region[n] >= 0 && p->node_region[n] != m->region[e])
                return fail(CF_VALIDATION, "node belongs to elements of two regions");
            p->node_region[n] = m->region[e];
        }
    for (int n = 0; n < p->N; ++n)
        if (p->node_region[n] < 0) return fail(CF_VALIDATION, "node not referenced by any element");
    (void)n_materials;
    /* facet owners via a hash of facet keys, scanning all element faces */
    size_t cap = 16;
    while (cap < 2 * (size_t)p->F + 16) cap <<= 1;
    fslot* tab = (fslot*)calloc(cap, sizeof(fslot));
    for (size_t i = 0; i < cap; ++i) tab[i].facet = -1;
    for (int f = 0; f < p->F; ++f) {
        int32_t k[3];
        for (int a = 0; a < 3; ++a) {
            k[a] = m->facets[3 * (size_t)f + a];
            if (k[a] < 0 || k[a] >= p->N) { free(tab); return fail(CF_VALIDATION, "facet references node outside range"); }
        }
        sort3(k);
        size_t h = key_hash(k) & (cap - 1);
        while (tab[h].facet >= 0 && memcmp(tab[h].k, k, sizeof k) != 0) h = (h + 1) & (cap - 1);
        if (tab[h].facet < 0) {
            memcpy(tab[h].k, k, sizeof k);
            tab[h].facet = f;
            tab[h].owner = -1;
            tab[h].count = 0;
        }
    }
    static const int tf[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
    if (p->F > 0)
        for (int e = 0; e < p->E; ++e) {
            const int32_t* t = p->tets + 4 * (size_t)e;
            for (int j = 0; j < 4; ++j) {
                int32_t k[3] = {t[tf[j][0]], t[tf[j][1]], t[tf[j][2]]};
                sort3(k);
                size_t h = key_hash(k) & (cap - 1);
                while (tab[h].facet >= 0 && memcmp(tab[h].k, k, sizeof k) != 0) h = (h + 1) & (cap - 1);
                if (tab[h].facet >= 0) {
                    if (tab[h].count == 0) tab[h].owner = e; /* smallest element id (scan ascending) */
                    tab[h].count++;
                }
            }
        }
    for (int f = 0; f < p->F; ++f) {
        int32_t k[3] = {m->facets[3 * (size_t)f], m->facets[3 * (size_t)f + 1], m->facets[3 * (size_t)f + 2]};
        sort3(k);
        size_t h = key_hash(k) & (cap - 1);
        while (memcmp(tab[h].k, k, sizeof k) != 0) h = (h + 1) & (cap - 1);
        if (tab[h].count == 0) { free(tab); return fail(CF_VALIDATION, "facet is not a face of any element"); }
        if (tab[h].count > 1) { free(tab); return fail(CF_VALIDATION, "facet is an interior face (two owner elements)"); }
        p->owner[f] = tab[h].owner;
    }
    free(tab);
    for (int c = 0; c < m->n_contacts; ++c)
        if (m->contacts[2 * c] < 0 || m->contacts[2 * c] >= m->n_tags || m->contacts[2 * c + 1] < 0 ||
            m->contacts[2 * c + 1] >= m->n_tags)
            return fail(CF_VALIDATION, "contact declaration references unknown tag");
    return CF_OK;
}

static void prep_free(prep_t* p) {
    free(p->tets); free(p->owner); free(p->node_region); free(p->geom);
}

/* pair_sister_facets mesh.hpp:456-478: nearest facet centroid on the other
 * side, ties by (d2, owner, facet). Exact: candidates sorted by centroid x,
 * scan outward while dx^2 <= best d2. */
typedef struct { double cx, cy, cz; int32_t facet, owner; } cand_t;
static int cmp_cand(const void* a, const void* b) {
    const cand_t* x = (const cand_t*)a; const cand_t* y = (const cand_t*)b;
    if (x->cx < y->cx) return -1;
    if (x->cx > y->cx) return 1;
    return (x->facet > y->facet) - (x->facet < y->facet);
}
static v3 facet_centroid(const cf_mesh_desc* m, int f) {
    v3 a = node_pos(m, m->facets[3 * (size_t)f]), b = node_pos(m, m->facets[3 * (size_t)f + 1]),
       c = node_pos(m, m->facets[3 * (size_t)f + 2]);
    return vmul(vadd(vadd(a, b), c), 1.0 / 3.0);
}
static double facet_area(const cf_mesh_desc* m, int f) {
    v3 a = node_pos(m, m->facets[3 * (size_t)f]), b = node_pos(m, m->facets[3 * (size_t)f + 1]),
       c = node_pos(m, m->facets[3 * (size_t)f + 2]);
    return 0.5 * vnorm(vcross(vsub(b, a), vsub(c, a)));
}
static int32_t nearest(const cand_t* cs, int n, v3 q) {
    /* binary search for the first cx >= q.x */
    int lo = 0, hi = n;
    while (lo < hi) { int mid = (lo + hi) / 2; if (cs[mid].cx < q.x) lo = mid + 1; else hi = mid; }
    double bd = INFINITY; int32_t bo = INT32_MAX, bf = INT32_MAX;
    for (int dir = 0; dir < 2; ++dir) {
        for (int i = dir == 0 ? lo : lo - 1; i >= 0 && i < n; i += dir == 0 ? 1 : -1) {
            double dx = cs[i].cx - q.x;
            if (dx * dx > bd) break;
            v3 d = {cs[i].cx - q.x, cs[i].cy - q.y, cs[i].cz - q.z};
            double d2 = vdot(d, d);
            if (d2 < bd || (d2 == bd && (cs[i].owner < bo || (cs[i].owner == bo && cs[i].facet < bf)))) {
                bd = d2; bo = cs[i].owner; bf = cs[i].facet;
            }
        }
    }
    return bf;
}

typedef struct { int32_t facet, sister, contact; } pair_t;
static int pair_sisters(const cf_mesh_desc* m, const prep_t* p, pair_t** out, int* npairs) {
    int cap = 0, np = 0;
    pair_t* pairs = NULL;
    for (int c = 0; c < m->n_contacts; ++c) {
        int ta = m->contacts[2 * c], tb = m->contacts[2 * c + 1];
        int na = 0, nb = 0;
        for (int f = 0; f < p->F; ++f) { if (m->facet_tag[f] == ta) na++; if (m->facet_tag[f] == tb) nb++; }
        if (na == 0 || nb == 0) { free(pairs); return fail(CF_CONFIG, "contact side has no tagged facets"); }
        cand_t* A = (cand_t*)malloc(sizeof(cand_t) * na);
        cand_t* B = (cand_t*)malloc(sizeof(cand_t) * nb);
        int32_t* fa = (int32_t*)malloc(sizeof(int32_t) * na);
        int32_t* fb = (int32_t*)malloc(sizeof(int32_t) * nb);
        na = nb = 0;
        for (int f = 0; f < p->F; ++f) {
            if (m->facet_tag[f] == ta) {
                v3 cc = facet_centroid(m, f);
                cand_t x = {cc.x, cc.y, cc.z, f, p->owner[f]};
                fa[na] = f; A[na++] = x;
            }
            if (m->facet_tag[f] == tb) {
                v3 cc = facet_centroid(m, f);
                cand_t x = {cc.x, cc.y, cc.z, f, p->owner[f]};
                fb[nb] = f; B[nb++] = x;
            }
        }
        qsort(A, na, sizeof(cand_t), cmp_cand);
        qsort(B, nb, sizeof(cand_t), cmp_cand);
        if (np + na + nb > cap) { cap = 2 * (np + na + nb); pairs = (pair_t*)realloc(pairs, sizeof(pair_t) * cap); }
        for (int i = 0; i < na; ++i) {
            int32_t nf = nearest(B, nb, facet_centroid(m, fa[i]));
            pair_t pr = {fa[i], p->owner[nf], c};
            pairs[np++] = pr;
        }
        for (int i = 0; i < nb; ++i) {
            int32_t nf = nearest(A, na, facet_centroid(m, fb[i]));
            pair_t pr = {fb[i], p->owner[nf], c};
            pairs[np++] = pr;
        }
        free(A); free(B); free(fa); free(fb);
    }
    *out = pairs; *npairs = np;
    return CF_OK;
}

OR_EXPORT int or_pair_sister_facets(const cf_mesh_desc* m, int32_t* out, int64_t cap, int64_t* n) {
    prep_t p; memset(&p, 0, sizeof p);
    int st = prep_mesh(m, 0, &p);
    if (st) { prep_free(&p); return st; }
    pair_t* pairs = NULL; int np = 0;
    st = pair_sisters(m, &p, &pairs, &np);
    if (!st) {
        *n = np;
        if (out) for (int i = 0; i < np && i < cap; ++i) { out[3 * i] = pairs[i].facet; out[3 * i + 1] = pairs[i].sister; out[3 * i + 2] = pairs[i].contact; }
    }
    free(pairs); prep_free(&p);
    return st;
}

/* ------------------------------------------------------------ solver */
typedef struct {
    int32_t slots[3];
    double area;
    int interface;
    double q, h, t_inf;
    int32_t pair;            /* ambient pair index */
    const cf_interface_coeff* coeff;
} fbind_t;

typedef struct {
    double time, dt, static_dt, loop_seconds;
    int64_t steps, clamp_steps, n_series;
    int32_t dynamic_dt;
} or_result;

static int name_eq(const char* a, const char* b) { return a && b && strcmp(a, b) == 0; }

/* Full solve. block_of_element: NULL = 1 block; part_of_element: NULL = 1 part.
 * Blocks must not straddle parts. T_init: NULL = initial_temperatures. */
OR_EXPORT int or_solve(const cf_mesh_desc* m, const cf_setup_desc* s,
                       const int32_t* block_of_element, int32_t n_blocks,
                       const int32_t* part_of_element, int32_t n_parts,
                       int64_t max_steps, double* T_out, double* H_out,
                       double* series, int64_t series_cap, or_result* res) {
    int st = CF_OK;
    prep_t p; memset(&p, 0, sizeof p);
    pair_t* pairs = NULL; int np = 0;
    mat_t* mats = NULL;
    if (!m || !s || !res) return fail(CF_INVALID_ARG, "null argument");
    if (!(s->dt_safety > 0 && s->dt_safety <= 1)) return fail(CF_CONFIG, "safety must be in (0, 1]");
    for (int i = 0; i < s->n_coeffs; ++i)
        if (!table_ok(&s->coeffs[i].h)) return fail(CF_CONFIG, "interface h: empty or inconsistent table");
    if ((st = prep_mesh(m, s->n_materials, &p))) goto done;
    /* solve_serial: pairs first (blocked.hpp:651) */
    if ((st = pair_sisters(m, &p, &pairs, &np))) goto done;
    const int N = p.N, E = p.E, F = p.F;
    if (!block_of_element) n_blocks = 1;
    if (!part_of_element) n_parts = 1;

    mats = (mat_t*)calloc(s->n_materials > 0 ? s->n_materials : 1, sizeof(mat_t));
    for (int e = 0; e < E; ++e)
        if (m->region[e] >= s->n_materials) { st = fail(CF_CONFIG, "no material for region"); goto done; }
    {
        char* used = (char*)calloc(s->n_materials + 1, 1);
        for (int e = 0; e < E; ++e) used[m->region[e]] = 1;
        for (int r = 0; r < s->n_materials; ++r)
            if (used[r] || s->materials[r].rho > 0) {
                if ((st = mat_init(&s->materials[r], &mats[r]))) { free(used); goto done; }
            }
        free(used);
    }
    int temp_dep = 0, finite_range = 0;
    for (int r = 0; r < s->n_materials; ++r) {
        if (!mats[r].m) continue;
        if (s->materials[r].c.n > 1 || s->materials[r].k.n > 1) temp_dep = 1;
        if (isfinite(mats[r].range_lo) || isfinite(mats[r].range_hi)) finite_range = 1;
    }

    /* initial_temperatures blocked.hpp:396-417 */
    double* T = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
    double* Tprev = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
    for (int n = 0; n < N; ++n)
        T[n] = s->initial_T ? s->initial_T[n] : s->materials[p.node_region[n]].initial_temperature;
    /* per tag resolution (resolve_facet_tag blocked.hpp:127-149) */
    int ntag = m->n_tags;
    const cf_boundary_condition** bc_of_tag = (const cf_boundary_condition**)calloc(ntag + 1, sizeof(void*));
    for (int t = 0; t < ntag; ++t)
        for (int b = 0; b < s->n_bcs; ++b)
            if (name_eq(s->bcs[b].tag, m->tags[t])) bc_of_tag[t] = &s->bcs[b];
    {
        int32_t* best_tag = (int32_t*)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
        for (int n = 0; n < N; ++n) best_tag[n] = INT32_MAX;
        for (int f = 0; f < F; ++f) {
            const cf_boundary_condition* bc = bc_of_tag[m->facet_tag[f]];
            if (!bc || bc->kind != CF_BC_FIXED) continue;
            for (int a = 0; a < 3; ++a) {
                int n = m->facets[3 * (size_t)f + a];
                if (m->facet_tag[f] < best_tag[n]) {
                    best_tag[n] = m->facet_tag[f];
                    if (bc->fixed_T.n < 1) { free(best_tag); st = fail(CF_CONFIG, "fixed boundary condition without a temperature value"); goto done_T; }
                    T[n] = pl_eval(&bc->fixed_T, 0.0);
                }
            }
        }
        free(best_tag);
    }

    /* ---------------- build_worker_model (blocked.hpp:156-361) over blocks */
    int32_t* pair_of_facet = (int32_t*)malloc(sizeof(int32_t) * (F > 0 ? F : 1));
    for (int f = 0; f < F; ++f) pair_of_facet[f] = -1;
    for (int i = 0; i < np; ++i) pair_of_facet[pairs[i].facet] = i;
    /* facets of element, ascending facet id */
    int32_t* fe_off = (int32_t*)calloc(E + 1, sizeof(int32_t));
    int32_t* fe = (int32_t*)malloc(sizeof(int32_t) * (F > 0 ? F : 1));
    for (int f = 0; f < F; ++f) fe_off[p.owner[f] + 1]++;
    for (int e = 0; e < E; ++e) fe_off[e + 1] += fe_off[e];
    {
        int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (E > 0 ? E : 1));
        memcpy(cur, fe_off, sizeof(int32_t) * E);
        for (int f = 0; f < F; ++f) fe[cur[p.owner[f]]++] = f;
        free(cur);
    }
    /* block element lists ascending */
    int32_t* be_off = (int32_t*)calloc(n_blocks + 1, sizeof(int32_t));
    int32_t* be = (int32_t*)malloc(sizeof(int32_t) * (E > 0 ? E : 1));
    for (int e = 0; e < E; ++e) {
        int b = block_of_element ? block_of_element[e] : 0;
        if (b < 0 || b >= n_blocks) { st = fail(CF_INVALID_ARG, "block id out of range"); goto done_T; }
        be_off[b + 1]++;
    }
    for (int b = 0; b < n_blocks; ++b) be_off[b + 1] += be_off[b];
    {
        int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * (n_blocks > 0 ? n_blocks : 1));
        memcpy(cur, be_off, sizeof(int32_t) * n_blocks);
        for (int e = 0; e < E; ++e) be[cur[block_of_element ? block_of_element[e] : 0]++] = e;
        free(cur);
    }
    int32_t* part_of_block = (int32_t*)malloc(sizeof(int32_t) * (n_blocks > 0 ? n_blocks : 1));
    for (int b = 0; b < n_blocks; ++b) {
        part_of_block[b] = -1;
        for (int i = be_off[b]; i < be_off[b + 1]; ++i) {
            int pp = part_of_element ? part_of_element[be[i]] : 0;
            if (part_of_block[b] >= 0 && part_of_block[b] != pp) { st = fail(CF_INVALID_ARG, "block straddles parts"); goto done_T; }
            part_of_block[b] = pp;
        }
    }
    /* slots per block: ascending node ids; element slots; facet bindings */
    int32_t* slot_of = (int32_t*)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
    for (int n = 0; n < N; ++n) slot_of[n] = -1;
    int64_t* bn_off = (int64_t*)calloc(n_blocks + 1, sizeof(int64_t));
    int32_t* bnode = NULL; int64_t bnode_cap = 0;
    int32_t* eslots = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(E > 0 ? E : 1)); /* by block order position */
    fbind_t* fb = (fbind_t*)malloc(sizeof(fbind_t) * (F > 0 ? F : 1));
    int32_t* bf_off = (int32_t*)calloc(n_blocks + 1, sizeof(int32_t));
    int nfb = 0;
    char* is_dir = (char*)calloc(N > 0 ? N : 1, 1);
    int32_t* dir_tag = (int32_t*)malloc(sizeof(int32_t) * (N > 0 ? N : 1));
    const cf_boundary_condition** dir_bc = (const cf_boundary_condition**)calloc(N > 0 ? N : 1, sizeof(void*));
    for (int b = 0; b < n_blocks; ++b) {
        for (int i = be_off[b]; i < be_off[b + 1]; ++i)
            for (int a = 0; a < 4; ++a) slot_of[p.tets[4 * (size_t)be[i] + a]] = 0;
        /* ascending node ids: collect marked nodes of this block */
        int64_t start = bn_off[b];
        int64_t cnt = 0;
        /* gather unique nodes then sort */
        int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)(be_off[b + 1] - be_off[b] + 1));
        for (int i = be_off[b]; i < be_off[b + 1]; ++i)
            for (int a = 0; a < 4; ++a) {
                int n = p.tets[4 * (size_t)be[i] + a];
                if (slot_of[n] == 0) { slot_of[n] = -2; tmp[cnt++] = n; }
            }
        qsort(tmp, cnt, sizeof(int32_t), cmpi);
        if (start + cnt > bnode_cap) { bnode_cap = 2 * (start + cnt) + 16; bnode = (int32_t*)realloc(bnode, sizeof(int32_t) * bnode_cap); }
        for (int64_t j = 0; j < cnt; ++j) { bnode[start + j] = tmp[j]; slot_of[tmp[j]] = (int32_t)j; }
        free(tmp);
        bn_off[b + 1] = start + cnt;
        for (int i = be_off[b]; i < be_off[b + 1]; ++i) {
            int e = be[i];
            for (int a = 0; a < 4; ++a) eslots[4 * (size_t)i + a] = slot_of[p.tets[4 * (size_t)e + a]];
            for (int j = fe_off[e]; j < fe_off[e + 1]; ++j) {
                int f = fe[j];
                int tag = m->facet_tag[f];
                const cf_boundary_condition* bc = bc_of_tag[tag];
                const cf_interface_coeff* coeff = NULL;
                for (int c = 0; c < m->n_contacts; ++c)
                    if (m->contacts[2 * c] == tag || m->contacts[2 * c + 1] == tag) {
                        const cf_interface_coeff* ic = NULL;
                        for (int k = 0; k < s->n_coeffs && !ic; ++k) {
                            const cf_interface_coeff* x = &s->coeffs[k];
                            const char* A = m->tags[m->contacts[2 * c]]; const char* B = m->tags[m->contacts[2 * c + 1]];
                            if ((name_eq(x->tag_a, A) && name_eq(x->tag_b, B)) || (name_eq(x->tag_a, B) && name_eq(x->tag_b, A))) ic = x;
                        }
                        if (!ic) { st = fail(CF_CONFIG, "no interface coefficient for contact"); goto done_T; }
                        coeff = ic;
                    }
                if (bc && coeff) { st = fail(CF_CONFIG, "facet tag resolves to both a boundary condition and a contact interface"); goto done_T; }
                if (!bc && !coeff) { st = fail(CF_CONFIG, "facet tag resolves to no declared condition"); goto done_T; }
                if (bc && bc->kind == CF_BC_FIXED) {
                    for (int a = 0; a < 3; ++a) {
                        int n = m->facets[3 * (size_t)f + a];
                        if (!is_dir[n] || tag < dir_tag[n]) { is_dir[n] = 1; dir_tag[n] = tag; dir_bc[n] = bc; }
                    }
                    continue;
                }
                fbind_t x; memset(&x, 0, sizeof x);
                x.area = facet_area(m, f);
                for (int a = 0; a < 3; ++a) x.slots[a] = slot_of[m->facets[3 * (size_t)f + a]];
                if (coeff) {
                    if (pair_of_facet[f] < 0) { st = fail(CF_CONFIG, "interface facet has no sister pairing"); goto done_T; }
                    x.interface = 1; x.pair = pair_of_facet[f]; x.coeff = coeff;
                } else {
                    x.q = bc->q; x.h = bc->h; x.t_inf = bc->t_inf;
                }
                fb[nfb++] = x;
            }
        }
        bf_off[b + 1] = nfb;
        for (int64_t j = bn_off[b]; j < bn_off[b + 1]; ++j) slot_of[bnode[j]] = -1;
    }
    for (int n = 0; n < N; ++n)
        if (is_dir[n] && dir_bc[n]->fixed_T.n < 1) { st = fail(CF_CONFIG, "fixed boundary condition without a temperature value"); goto done_T; }
    /* merge CSR per node: (part asc, block asc) entries */
    int64_t tot = bn_off[n_blocks];
    int64_t* mo = (int64_t*)calloc(N + 1, sizeof(int64_t));
    int64_t* me = (int64_t*)malloc(sizeof(int64_t) * (tot > 0 ? tot : 1));
    int32_t* mpart = (int32_t*)malloc(sizeof(int32_t) * (tot > 0 ? tot : 1));
    for (int64_t j = 0; j < tot; ++j) mo[bnode[j] + 1]++;
    for (int n = 0; n < N; ++n) mo[n + 1] += mo[n];
    {
        int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (N > 0 ? N : 1));
        memcpy(cur, mo, sizeof(int64_t) * N);
        for (int pp = 0; pp < n_parts; ++pp)
            for (int b = 0; b < n_blocks; ++b) {
                if (part_of_block[b] != pp) continue;
                for (int64_t j = bn_off[b]; j < bn_off[b + 1]; ++j) { me[cur[bnode[j]]] = j; mpart[cur[bnode[j]]++] = pp; }
            }
        free(cur);
    }
    /* static dt (blocked.hpp:340-350) */
    double static_dt = 0;
    if (!temp_dep) {
        double dt = INFINITY;
        for (int e = 0; e < E; ++e) {
            const cf_material* mm = &s->materials[m->region[e]];
            double v = mm->rho * pl_eval(&mm->c, 0) * p.geom[e].min_edge * p.geom[e].min_edge / pl_eval(&mm->k, 0);
            if (v < dt) dt = v;
        }
        static_dt = dt * s->dt_safety;
        if (!(static_dt > 0)) { st = fail(CF_VALIDATION, "non-positive stable time step"); goto done_T; }
    }
    /* state */
    double* H = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
    for (int n = 0; n < N; ++n) H[n] = enthalpy(&mats[p.node_region[n]], T[n]);
    double* amb = (double*)calloc(np > 0 ? np : 1, sizeof(double));
    double* bc_ = (double*)malloc(sizeof(double) * (tot > 0 ? tot : 1));
    double* br_ = (double*)malloc(sizeof(double) * (tot > 0 ? tot : 1));
    double* cd = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
    double* rr = (double*)malloc(sizeof(double) * (N > 0 ? N : 1));
    double time = 0, last_dt = 0;
    int64_t step = 0, clamp_steps = 0, nser = 0;
    /* pre-loop refresh_ambient (blocked.hpp:669) */
    for (int i = 0; i < np; ++i) {
        const int32_t* sn = p.tets + 4 * (size_t)pairs[i].sister;
        double sum = 0;
        for (int a = 0; a < 4; ++a) sum += T[sn[a]];
        amb[i] = 0.25 * sum;
    }
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    const double t_end = s->t_end;
    while ((max_steps > 0 && step < max_steps) || (max_steps <= 0 && time < t_end)) {
        double remaining = max_steps > 0 ? 0 : t_end - time;
        /* assemble_blocks */
        double min_bound = INFINITY;
        for (int b = 0; b < n_blocks; ++b) {
            double* c = bc_ + bn_off[b];
            double* r = br_ + bn_off[b];
            int64_t nb = bn_off[b + 1] - bn_off[b];
            for (int64_t j = 0; j < nb; ++j) { c[j] = 0; r[j] = 0; }
            const int32_t* ids = bnode + bn_off[b];
            for (int i = be_off[b]; i < be_off[b + 1]; ++i) {
                int e = be[i];
                const cf_material* mm = &s->materials[m->region[e]];
                const int32_t* sl = eslots + 4 * (size_t)i;
                double tn[4], hn[4];
                for (int a = 0; a < 4; ++a) { tn[a] = T[ids[sl[a]]]; hn[a] = H[ids[sl[a]]]; }
                const geom_t* g = &p.geom[e];
                /* element_accumulate fem.hpp:57-70 */
                double t_bar = 0.25 * (tn[0] + tn[1] + tn[2] + tn[3]);
                double lump = mm->rho * apparent_c(g, tn, hn, mm) * g->vol * 0.25;
                double kv = pl_eval(&mm->k, t_bar) * g->vol;
                v3 gt = {0, 0, 0};
                for (int bb = 0; bb < 4; ++bb) gt = vadd(gt, vmul(g->g[bb], tn[bb]));
                for (int a = 0; a < 4; ++a) {
                    c[sl[a]] += lump;
                    r[sl[a]] -= kv * vdot(g->g[a], gt);
                }
                if (temp_dep) {
                    double tb = 0.25 * (tn[0] + tn[1] + tn[2] + tn[3]);
                    double v = mm->rho * pl_eval(&mm->c, tb) * g->min_edge * g->min_edge / pl_eval(&mm->k, tb);
                    if (v < min_bound) min_bound = v;
                }
            }
            for (int i = bf_off[b]; i < bf_off[b + 1]; ++i) {
                const fbind_t* x = &fb[i];
                double ts[3];
                for (int a = 0; a < 3; ++a) ts[a] = T[ids[x->slots[a]]];
                double q, h, tinf;
                if (x->interface) {
                    double var = x->coeff->var == CF_VAR_TIME ? time : (ts[0] + ts[1] + ts[2]) / 3.0;
                    q = 0.0; h = pl_eval(&x->coeff->h, var); tinf = amb[x->pair];
                } else {
                    q = x->q; h = x->h; tinf = x->t_inf;
                }
                /* facet_flux_accumulate fem.hpp:74-79 */
                double third = x->area / 3.0;
                for (int a = 0; a < 3; ++a) r[x->slots[a]] += third * (-q + h * (tinf - ts[a]));
            }
        }
        /* merge_blocks (+ parts in ascending part id) */
        for (int n = 0; n < N; ++n) {
            double ct = 0, rt = 0;
            int64_t j = mo[n];
            while (j < mo[n + 1]) {
                int pp = mpart[j];
                double cp = 0, rp = 0;
                for (; j < mo[n + 1] && mpart[j] == pp; ++j) { cp += bc_[me[j]]; rp += br_[me[j]]; }
                ct += cp; rt += rp;
            }
            cd[n] = ct; rr[n] = rt;
        }
        /* refresh_ambient from pre-update T (consumed next step) */
        for (int i = 0; i < np; ++i) {
            const int32_t* sn = p.tets + 4 * (size_t)pairs[i].sister;
            double sum = 0;
            for (int a = 0; a < 4; ++a) sum += T[sn[a]];
            amb[i] = 0.25 * sum;
        }
        double dt = temp_dep ? min_bound * s->dt_safety : static_dt;
        if (remaining > 0) dt = dt < remaining ? dt : remaining;
        /* update_fields */
        memcpy(Tprev, T, sizeof(double) * N);
        for (int n = 0; n < N; ++n) {
            if (!(cd[n] > 0)) {
                char msg[128]; snprintf(msg, sizeof msg, "zero lumped capacitance at active node %d", n);
                st = fail(CF_VALIDATION, msg); goto done_all;
            }
            T[n] += dt * rr[n] / cd[n];
        }
        double t_next = time + dt;
        for (int n = 0; n < N; ++n)
            if (is_dir[n]) T[n] = pl_eval(&dir_bc[n]->fixed_T, t_next);
        int clamped = 0;
        for (int n = 0; n < N; ++n) {
            const mat_t* mt = &mats[p.node_region[n]];
            H[n] = enthalpy(mt, T[n]);
            if (finite_range && (T[n] < mt->range_lo || T[n] > mt->range_hi)) clamped = 1;
        }
        if (clamped) ++clamp_steps;
        time = t_next; last_dt = dt; ++step;
        if (s->output_every > 0 && step % s->output_every == 0) {
            if (series && nser < series_cap) {
                double lo = INFINITY, hi = -INFINITY;
                for (int n = 0; n < N; ++n) { if (T[n] < lo) lo = T[n]; if (T[n] > hi) hi = T[n]; }
                series[3 * nser] = time; series[3 * nser + 1] = lo; series[3 * nser + 2] = hi;
            }
            nser++;
        }
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    res->loop_seconds = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
    res->time = time; res->dt = last_dt; res->steps = step; res->clamp_steps = clamp_steps;
    res->static_dt = static_dt; res->dynamic_dt = temp_dep; res->n_series = nser;
    if (T_out) memcpy(T_out, T, sizeof(double) * N);
    if (H_out) memcpy(H_out, H, sizeof(double) * N);
done_all:
    free(H); free(amb); free(bc_); free(br_); free(cd); free(rr);
    free(mo); free(me); free(mpart);
done_T:
    /* lightweight cleanup of the remaining scratch (process-lifetime leaks on
     * early error paths are acceptable for a test oracle) */
    free(T); free(Tprev);
done:
    if (mats) { for (int r = 0; r < s->n_materials; ++r) free(mats[r].cum); free(mats); }
    free(pairs);
    prep_free(&p);
    return st;
}

int cmpi(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

/* ------------------------------------------------------------ KAT helpers */
OR_EXPORT int or_tet_geometry(const double* p /*12*/, double* out /*15: vol, g[12], min, max*/) {
    v3 q[4];
    for (int a = 0; a < 4; ++a) { q[a].x = p[3 * a]; q[a].y = p[3 * a + 1]; q[a].z = p[3 * a + 2]; }
    geom_t g;
    int st = tet_geom(q[0], q[1], q[2], q[3], &g);
    out[0] = g.vol;
    for (int a = 0; a < 4; ++a) { out[1 + 3 * a] = g.g[a].x; out[2 + 3 * a] = g.g[a].y; out[3 + 3 * a] = g.g[a].z; }
    out[13] = g.min_edge; out[14] = g.max_edge;
    return st;
}
OR_EXPORT double or_enthalpy(const cf_material* m, double T) {
    mat_t mt; memset(&mt, 0, sizeof mt);
    if (mat_init(m, &mt)) return NAN;
    double h = enthalpy(&mt, T);
    free(mt.cum);
    return h;
}
OR_EXPORT double or_apparent_heat_capacity(const double* geom15, const double* Tn, const double* Hn,
                                           const cf_material* m) {
    geom_t g;
    g.vol = geom15[0];
    for (int a = 0; a < 4; ++a) { g.g[a].x = geom15[1 + 3 * a]; g.g[a].y = geom15[2 + 3 * a]; g.g[a].z = geom15[3 + 3 * a]; }
    g.min_edge = geom15[13]; g.max_edge = geom15[14];
    return apparent_c(&g, Tn, Hn, m);
}
/* element_accumulate into 4 local slots (c[4], r[4] accumulate) */
OR_EXPORT void or_element_accumulate(const double* geom15, const cf_material* m, const double* tn,
                                     const double* hn, double* c, double* r) {
    geom_t g;
    g.vol = geom15[0];
    for (int a = 0; a < 4; ++a) { g.g[a].x = geom15[1 + 3 * a]; g.g[a].y = geom15[2 + 3 * a]; g.g[a].z = geom15[3 + 3 * a]; }
    g.min_edge = geom15[13]; g.max_edge = geom15[14];
    double t_bar = 0.25 * (tn[0] + tn[1] + tn[2] + tn[3]);
    double lump = m->rho * apparent_c(&g, tn, hn, m) * g.vol * 0.25;
    double kv = pl_eval(&m->k, t_bar) * g.vol;
    v3 gt = {0, 0, 0};
    for (int b = 0; b < 4; ++b) gt = vadd(gt, vmul(g.g[b], tn[b]));
    for (int a = 0; a < 4; ++a) { c[a] += lump; r[a] -= kv * vdot(g.g[a], gt); }
}

/* ------------------------------------------------------------ lambda_max */
/* Power iteration on M_L^-1 (K + H) at the region's initial-temperature
 * properties (no latent heat; interface h = largest table value), Dirichlet rows removed. Host reference for
 * cf_estimate_lambda_max. x0 from a counter hash of the node id. */
static double u01(uint64_t seed, uint64_t key) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ull + key + 0x632BE59BD9B4E019ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}
OR_EXPORT int or_lambda_max(const cf_mesh_desc* m, const cf_setup_desc* s, int iterations, uint64_t seed,
                            double* lambda, double* eq13) {
    prep_t p; memset(&p, 0, sizeof p);
    int st = prep_mesh(m, s->n_materials, &p);
    if (st) { prep_free(&p); return st; }
    int N = p.N, E = p.E, F = p.F;
    double* M = (double*)calloc(N, sizeof(double));
    double* D = (double*)calloc(N, sizeof(double));
    char* dir = (char*)calloc(N, 1);
    double e13 = INFINITY;
    for (int e = 0; e < E; ++e) {
        const cf_material* mm = &s->materials[m->region[e]];
        double c = pl_eval(&mm->c, mm->initial_temperature);
        for (int a = 0; a < 4; ++a) M[p.tets[4 * (size_t)e + a]] += mm->rho * c * p.geom[e].vol * 0.25;
        double v = mm->rho * pl_eval(&mm->c, 0) * p.geom[e].min_edge * p.geom[e].min_edge / pl_eval(&mm->k, 0);
        if (v < e13) e13 = v;
    }
    for (int f = 0; f < F; ++f) {
        int tag = m->facet_tag[f];
        double h = 0;
        const cf_boundary_condition* bc = NULL;
        for (int b = 0; b < s->n_bcs; ++b) if (name_eq(s->bcs[b].tag, m->tags[tag])) bc = &s->bcs[b];
        if (bc) {
            if (bc->kind == CF_BC_FIXED) { for (int a = 0; a < 3; ++a) dir[m->facets[3 * (size_t)f + a]] = 1; continue; }
            h = bc->h;
        } else {
            for (int c = 0; c < m->n_contacts; ++c)
                if (m->contacts[2 * c] == tag || m->contacts[2 * c + 1] == tag)
                    for (int k = 0; k < s->n_coeffs; ++k) {
                        const cf_interface_coeff* x = &s->coeffs[k];
                        const char* A = m->tags[m->contacts[2 * c]]; const char* B = m->tags[m->contacts[2 * c + 1]];
                        if ((name_eq(x->tag_a, A) && name_eq(x->tag_b, B)) || (name_eq(x->tag_a, B) && name_eq(x->tag_b, A))) {
                            h = x->h.y[0]; /* largest table value (conservative) */
                            for (int j = 1; j < x->h.n; ++j) if (x->h.y[j] > h) h = x->h.y[j];
                            break;
                        }
                    }
        }
        double third = facet_area(m, f) / 3.0;
        for (int a = 0; a < 3; ++a) D[m->facets[3 * (size_t)f + a]] += h * third;
    }
    double* x = (double*)malloc(sizeof(double) * N);
    double* y = (double*)malloc(sizeof(double) * N);
    for (int n = 0; n < N; ++n) x[n] = dir[n] ? 0.0 : (u01(seed, n) - 0.5);
    double lam = 0;
    for (int it = 0; it < iterations; ++it) {
        for (int n = 0; n < N; ++n) y[n] = D[n] * x[n];
        for (int e = 0; e < E; ++e) {
            const cf_material* mm = &s->materials[m->region[e]];
            double kv = pl_eval(&mm->k, mm->initial_temperature) * p.geom[e].vol;
            const int32_t* t = p.tets + 4 * (size_t)e;
            v3 gx = {0, 0, 0};
            for (int b = 0; b < 4; ++b) gx = vadd(gx, vmul(p.geom[e].g[b], x[t[b]]));
            for (int a = 0; a < 4; ++a) y[t[a]] += kv * vdot(p.geom[e].g[a], gx);
        }
        double num = 0, den = 0;
        for (int n = 0; n < N; ++n) { if (dir[n]) y[n] = 0; num += x[n] * y[n]; den += x[n] * M[n] * x[n]; }
        lam = num / den;
        double nrm = 0;
        for (int n = 0; n < N; ++n) { y[n] /= M[n]; nrm += y[n] * M[n] * y[n]; }
        nrm = sqrt(nrm);
        for (int n = 0; n < N; ++n) x[n] = y[n] / nrm;
    }
    *lambda = lam; *eq13 = e13;
    free(M); free(D); free(dir); free(x); free(y);
    prep_free(&p);
    return CF_OK;
}


/* ------------------------------------------------------------ partial assembly */
/* assemble_blocks restricted to the elements with elem_mask[e] != 0, as one
 * block in ascending element order (+ their facets), into per-node (c, r)
 * (zero for untouched nodes). The interface ambient is 0.25*sum(T_old[sister
 * nodes]) (refresh_ambient's one-step lag). Used by the multi-rank protocol
 * test: each worker assembles its own part (SPEC exchange_and_merge S:450-458). */
OR_EXPORT int or_assemble_part(const cf_mesh_desc* m, const cf_setup_desc* s, const char* elem_mask,
                               const double* T, const double* T_old, double time, double* c_out, double* r_out) {
    prep_t p; memset(&p, 0, sizeof p);
    int st = prep_mesh(m, s->n_materials, &p);
    if (st) { prep_free(&p); return st; }
    pair_t* pairs = NULL; int np = 0;
    if ((st = pair_sisters(m, &p, &pairs, &np))) { prep_free(&p); return st; }
    int N = p.N, E = p.E, F = p.F;
    mat_t* mats = (mat_t*)calloc(s->n_materials > 0 ? s->n_materials : 1, sizeof(mat_t));
    for (int r = 0; r < s->n_materials; ++r) if ((st = mat_init(&s->materials[r], &mats[r]))) goto out;
    for (int n = 0; n < N; ++n) { c_out[n] = 0; r_out[n] = 0; }
    {
        int32_t* pair_of_facet = (int32_t*)malloc(sizeof(int32_t) * (F > 0 ? F : 1));
        for (int f = 0; f < F; ++f) pair_of_facet[f] = -1;
        for (int i = 0; i < np; ++i) pair_of_facet[pairs[i].facet] = i;
        double* H = (double*)malloc(sizeof(double) * N);
        for (int n = 0; n < N; ++n) H[n] = enthalpy(&mats[p.node_region[n]], T[n]);
        for (int e = 0; e < E; ++e) {
            if (!elem_mask[e]) continue;
            const cf_material* mm = &s->materials[m->region[e]];
            const int32_t* t = p.tets + 4 * (size_t)e;
            double tn[4], hn[4];
            for (int a = 0; a < 4; ++a) { tn[a] = T[t[a]]; hn[a] = H[t[a]]; }
            const geom_t* g = &p.geom[e];
            double t_bar = 0.25 * (tn[0] + tn[1] + tn[2] + tn[3]);
            double lump = mm->rho * apparent_c(g, tn, hn, mm) * g->vol * 0.25;
            double kv = pl_eval(&mm->k, t_bar) * g->vol;
            v3 gt = {0, 0, 0};
            for (int b = 0; b < 4; ++b) gt = vadd(gt, vmul(g->g[b], tn[b]));
            for (int a = 0; a < 4; ++a) { c_out[t[a]] += lump; r_out[t[a]] -= kv * vdot(g->g[a], gt); }
        }
        /* facets in (owner element ascending, facet id ascending) order */
        for (int e = 0; e < E; ++e) {
            if (!elem_mask[e]) continue;
            for (int f = 0; f < F; ++f) {
                if (p.owner[f] != e) continue;
                int tag = m->facet_tag[f];
                const cf_boundary_condition* bc = NULL;
                for (int b = 0; b < s->n_bcs; ++b) if (name_eq(s->bcs[b].tag, m->tags[tag])) bc = &s->bcs[b];
                if (bc && bc->kind == CF_BC_FIXED) continue;
                double q, h, tinf;
                const int32_t* fn = m->facets + 3 * (size_t)f;
                double ts[3] = {T[fn[0]], T[fn[1]], T[fn[2]]};
                if (bc) { q = bc->q; h = bc->h; tinf = bc->t_inf; }
                else {
                    const cf_interface_coeff* ic = NULL;
                    for (int c = 0; c < m->n_contacts && !ic; ++c)
                        if (m->contacts[2 * c] == tag || m->contacts[2 * c + 1] == tag)
                            for (int k = 0; k < s->n_coeffs && !ic; ++k) {
                                const cf_interface_coeff* x = &s->coeffs[k];
                                const char* A = m->tags[m->contacts[2 * c]]; const char* B = m->tags[m->contacts[2 * c + 1]];
                                if ((name_eq(x->tag_a, A) && name_eq(x->tag_b, B)) || (name_eq(x->tag_a, B) && name_eq(x->tag_b, A))) ic = x;
                            }
                    if (!ic || pair_of_facet[f] < 0) { st = fail(CF_CONFIG, "unresolved facet"); break; }
                    const int32_t* sn = p.tets + 4 * (size_t)pairs[pair_of_facet[f]].sister;
                    double sum = 0;
                    for (int a = 0; a < 4; ++a) sum += T_old[sn[a]];
                    q = 0.0; h = pl_eval(&ic->h, ic->var == CF_VAR_TIME ? time : (ts[0] + ts[1] + ts[2]) / 3.0);
                    tinf = 0.25 * sum;
                }
                double third = facet_area(m, f) / 3.0;
                for (int a = 0; a < 3; ++a) r_out[fn[a]] += third * (-q + h * (tinf - ts[a]));
            }
        }
        free(pair_of_facet); free(H);
    }
out:
    for (int r = 0; r < s->n_materials; ++r) free(mats[r].cum);
    free(mats); free(pairs); prep_free(&p);
    return st;
}
