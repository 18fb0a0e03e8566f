// cf_plan.cpp — setup resolution and the tile (cache-block) builder.
//
// Reference semantics kept (paths relative to /root/reference/proj/include/castfem/):
//   MaterialTable::finalize / validate   material.hpp:40-47, 104-119; parse_config checks :339-344
//   resolve_facet_tag                    blocked.hpp:127-149
//   Dirichlet "lowest tag wins"          blocked.hpp:250-263, initial_temperatures :396-417
//   static dt (constant properties)      blocked.hpp:340-350, element_stable_dt fem.hpp:83-85
//   block-local slots + merge CSR        blocked.hpp:217-307 (tiles replace partition_graph blocks)
//   facet bindings in element order      blocked.hpp:244-288
//   external nodes / ambient bindings    blocked.hpp:309-331, classify_nodes partition.hpp:305-367
#include <omp.h>
#include <parallel/algorithm>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <array>
#include <map>
#include <numeric>

#include "cf_internal.hpp"
#include "cf_tilepack.hpp"

namespace cfb {

double pl_eval(const DevParams& P, const DevTable& t, double x) {
    const double* xs = P.pool + t.off;
    const double* ys = xs + t.n;
    if (t.n <= 1) return ys[0];
    if (x <= xs[0]) return ys[0];
    if (x >= xs[t.n - 1]) return ys[t.n - 1];
    int i = 0;
    while (i + 1 < t.n && xs[i + 1] <= x) ++i;
    const double f = (x - xs[i]) / (xs[i + 1] - xs[i]);
    return ys[i] + f * (ys[i + 1] - ys[i]);
}

double enthalpy(const DevParams& P, const DevMaterial& m, double T) {
    double sensible;
    if (m.c.n <= 1) {
        sensible = m.c0 * (T - m.ref);
    } else {
        const double* xs = P.pool + m.c.off;
        const double* ys = xs + m.c.n;
        const int n = m.c.n;
        const double Tc = T < xs[0] ? xs[0] : (xs[n - 1] < T ? xs[n - 1] : T);
        int ub = 0;
        while (ub < n && xs[ub] <= Tc) ++ub;
        const int i = std::min(ub, n - 1) - 1;
        sensible = P.pool[m.cum_off + i] + 0.5 * (ys[i] + pl_eval(P, m.c, Tc)) * (Tc - xs[i]);
    }
    double mf = 0;
    if (m.has_phase) {
        const double v = (T - m.solidus) / (m.liquidus - m.solidus);
        mf = v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
    }
    return sensible + m.latent * mf;
}

namespace {

struct Pool {
    DevParams& P;
    int used = 0;
    DevTable put(const cf_table& t, const char* what) {
        if (t.n < 1 || !t.x || !t.y) raise(CF_CONFIG, std::string(what) + ": empty or inconsistent table");
        for (int i = 1; i < t.n; ++i)
            if (!(t.x[i] > t.x[i - 1]))
                raise(CF_CONFIG, std::string(what) + ": table abscissae must be strictly increasing");
        if (used + 2 * t.n > kMaxTablePts) raise(CF_CONFIG, "tables exceed the device table pool");
        DevTable d{t.n, used};
        for (int i = 0; i < t.n; ++i) {
            P.pool[used + i] = t.x[i];
            P.pool[used + t.n + i] = t.y[i];
        }
        used += 2 * t.n;
        return d;
    }
};

bool name_eq(const char* a, const std::string& b) { return a && b == a; }

}  // namespace

void resolve_setup(const MeshData& m, const cf_setup_desc* s, SetupData& out) {
    resolve_setup_impl(m, s, out, nullptr, true);
}

void resolve_setup_impl(const MeshData& m, const cf_setup_desc* s, SetupData& out, const RegionUse* ru,
                        bool node_arrays) {
    if (!s) raise(CF_INVALID_ARG, "null setup");
    if ((s->n_materials && !s->materials) || (s->n_bcs && !s->bcs) || (s->n_coeffs && !s->coeffs))
        raise(CF_INVALID_ARG, "null array in setup descriptor");
    if (!(s->dt_safety > 0 && s->dt_safety <= 1)) raise(CF_CONFIG, "safety must be in (0, 1]");
    DevParams& P = out.P;
    std::memset(&P, 0, sizeof P);
    Pool pool{P};
    for (int i = 0; i < s->n_coeffs; ++i) {
        const cf_table& t = s->coeffs[i].h;
        if (t.n < 1 || !t.x || !t.y) raise(CF_CONFIG, "interface h: empty or inconsistent table");
        for (int j = 1; j < t.n; ++j)
            if (!(t.x[j] > t.x[j - 1])) raise(CF_CONFIG, "interface h: table abscissae must be strictly increasing");
    }
    // pair_sister_facets first (solve_serial blocked.hpp:651)
    trace_stage("resolve: tables");
    out.pairs = pair_sister_facets(m);
    trace_stage("resolve: sister pairing");
    out.pair_of_facet.assign(m.F, -1);
    for (size_t p = 0; p < out.pairs.size(); ++p) out.pair_of_facet[out.pairs[p].facet] = (int32_t)p;

    // materials of used regions (MaterialTable::finalize)
    std::vector<char> used(s->n_materials + 1, 0);
    if (!ru) {
        for (int32_t e = 0; e < m.E; ++e)
            if (m.region[e] >= s->n_materials)
                raise(CF_CONFIG, "no material for region " + std::to_string(m.region[e]));
        if (s->n_materials > kMaxRegions) raise(CF_CONFIG, "more than 16 material regions");
        for (int32_t e = 0; e < m.E; ++e) used[m.region[e]] = 1;
    } else {
        if (ru->first_bad_region >= 0) raise(CF_CONFIG, "no material for region " + std::to_string(ru->first_bad_region));
        if (s->n_materials > kMaxRegions) raise(CF_CONFIG, "more than 16 material regions");
        for (int r = 0; r < s->n_materials && r < 32; ++r) used[r] = (ru->mask >> r) & 1;
    }
    P.n_materials = s->n_materials;
    for (int r = 0; r < s->n_materials; ++r) {
        const cf_material& c = s->materials[r];
        DevMaterial& d = P.mat[r];
        if (!used[r] && !(c.rho > 0)) continue;  // untouched slot
        d.c = pool.put(c.c, "c");
        d.k = pool.put(c.k, "k");
        if (!(c.rho > 0)) raise(CF_CONFIG, "rho must be positive");
        for (int i = 0; i < c.c.n; ++i)
            if (c.c.y[i] <= 0) raise(CF_CONFIG, "c(T) must be positive");
        for (int i = 0; i < c.k.n; ++i)
            if (c.k.y[i] <= 0) raise(CF_CONFIG, "k(T) must be positive");
        if (c.latent_heat < 0) raise(CF_CONFIG, "latent_heat must be non-negative");
        if (c.latent_heat > 0 && !(c.solidus < c.liquidus))
            raise(CF_CONFIG, "phase change requires solidus < liquidus");
        d.rho = c.rho;
        d.T0 = c.initial_temperature;
        d.latent = c.latent_heat;
        d.solidus = c.solidus;
        d.liquidus = c.liquidus;
        d.has_phase = c.latent_heat > 0;
        d.c0 = c.c.y[0];
        d.k0 = c.k.y[0];
        d.ref = c.c.n <= 1 ? 0.0 : c.c.x[0];
        const int nc = std::max(c.c.n, 1);
        if (pool.used + nc > kMaxTablePts) raise(CF_CONFIG, "tables exceed the device table pool");
        d.cum_off = pool.used;
        P.pool[d.cum_off] = 0;
        for (int i = 1; i < c.c.n; ++i)
            P.pool[d.cum_off + i] =
                P.pool[d.cum_off + i - 1] + 0.5 * (c.c.y[i] + c.c.y[i - 1]) * (c.c.x[i] - c.c.x[i - 1]);
        pool.used += nc;
        d.range_lo = -INFINITY;
        d.range_hi = INFINITY;
        if (c.c.n > 1) d.range_lo = std::max(d.range_lo, c.c.x[0]);
        if (c.k.n > 1) d.range_lo = std::max(d.range_lo, c.k.x[0]);
        if (c.c.n > 1) d.range_hi = std::min(d.range_hi, c.c.x[c.c.n - 1]);
        if (c.k.n > 1) d.range_hi = std::min(d.range_hi, c.k.x[c.k.n - 1]);
        if (c.c.n > 1 || c.k.n > 1) P.temp_dep = 1;
        if (std::isfinite(d.range_lo) || std::isfinite(d.range_hi)) P.finite_range = 1;
    }
    out.temp_dep = P.temp_dep != 0;
    P.dt_safety = s->dt_safety;

    // boundary conditions by tag name (map semantics: last declaration wins)
    const int32_t ntag = (int32_t)m.tags.size();
    std::vector<int32_t> bc_of_tag(ntag, -1);
    for (int32_t t = 0; t < ntag; ++t)
        for (int b = 0; b < s->n_bcs; ++b)
            if (name_eq(s->bcs[b].tag, m.tags[t])) bc_of_tag[t] = b;
    // interface coefficient per contact: first match (find_interface material.hpp:175-179)
    const int32_t nct = (int32_t)m.contacts.size() / 2;
    std::vector<int32_t> coeff_of_contact(nct, -1);
    for (int32_t c = 0; c < nct; ++c) {
        const std::string& A = m.tags[m.contacts[2 * c]];
        const std::string& B = m.tags[m.contacts[2 * c + 1]];
        for (int k = 0; k < s->n_coeffs && coeff_of_contact[c] < 0; ++k) {
            const cf_interface_coeff& x = s->coeffs[k];
            if ((name_eq(x.tag_a, A) && name_eq(x.tag_b, B)) || (name_eq(x.tag_a, B) && name_eq(x.tag_b, A)))
                coeff_of_contact[c] = k;
        }
    }
    // per tag resolution -> kind ids
    std::vector<int32_t> kind_of_tag(ntag, INT32_MIN);
    std::map<int32_t, int32_t> kind_of_bc, kind_of_coeff, dir_of_bc;
    std::vector<int32_t> tag_seen(ntag, 0);
    for (int32_t f = 0; f < m.F; ++f) tag_seen[m.facet_tag[f]] = 1;
    for (int32_t t = 0; t < ntag; ++t) {
        if (!tag_seen[t]) continue;
        const int32_t b = bc_of_tag[t];
        int32_t coeff = -1;
        for (int32_t c = 0; c < nct; ++c)
            if (m.contacts[2 * c] == t || m.contacts[2 * c + 1] == t) {
                if (coeff_of_contact[c] < 0)
                    raise(CF_CONFIG, "no interface coefficient for contact " + m.tags[m.contacts[2 * c]] + "/" +
                                         m.tags[m.contacts[2 * c + 1]]);
                coeff = coeff_of_contact[c];
            }
        if (b >= 0 && coeff >= 0)
            raise(CF_CONFIG, "facet tag '" + m.tags[t] + "' resolves to both a boundary condition and a contact interface");
        if (b < 0 && coeff < 0) raise(CF_CONFIG, "facet tag '" + m.tags[t] + "' resolves to no declared condition");
        if (b >= 0 && s->bcs[b].kind == CF_BC_FIXED) {
            if (!dir_of_bc.count(b)) {
                const int32_t id = (int32_t)dir_of_bc.size();
                if (id >= kMaxFacetKinds) raise(CF_CONFIG, "too many fixed boundary conditions");
                dir_of_bc[b] = id;
                const cf_table& ft = s->bcs[b].fixed_T;
                if (ft.n < 1) raise(CF_CONFIG, "fixed boundary condition without a temperature value");
                P.dir_tab[id] = pool.put(ft, "T");
            }
            kind_of_tag[t] = -1 - dir_of_bc[b];
        } else if (b >= 0) {
            if (!kind_of_bc.count(b)) {
                const int32_t id = P.n_kinds++;
                if (id >= kMaxFacetKinds) raise(CF_CONFIG, "too many facet conditions");
                kind_of_bc[b] = id;
                P.kind[id].interface = 0;
                P.kind[id].q = s->bcs[b].q;
                P.kind[id].h = s->bcs[b].h;
                P.kind[id].t_inf = s->bcs[b].t_inf;
            }
            kind_of_tag[t] = kind_of_bc[b];
        } else {
            if (!kind_of_coeff.count(coeff)) {
                const int32_t id = P.n_kinds++;
                if (id >= kMaxFacetKinds) raise(CF_CONFIG, "too many facet conditions");
                kind_of_coeff[coeff] = id;
                P.kind[id].interface = 1;
                P.kind[id].var = s->coeffs[coeff].var == CF_VAR_TEMPERATURE ? CF_VAR_TEMPERATURE : CF_VAR_TIME;
                P.kind[id].q = 0.0;
                P.kind[id].htab = pool.put(s->coeffs[coeff].h, "interface h");
            }
            kind_of_tag[t] = kind_of_coeff[coeff];
        }
    }
    out.kind_of_tag = kind_of_tag;
    out.facet_kind.resize(m.F);
    for (int32_t f = 0; f < m.F; ++f) {
        out.facet_kind[f] = kind_of_tag[m.facet_tag[f]];
        if (out.facet_kind[f] >= 0 && P.kind[out.facet_kind[f]].interface && out.pair_of_facet[f] < 0)
            raise(CF_CONFIG, "interface facet " + std::to_string(f) + " has no sister pairing; call pair_sister_facets");
    }
    if (!node_arrays) {
        out.static_dt_only = true;
    } else {
    // Dirichlet nodes: lowest tag wins
    out.dir_of_node.assign(m.N, -1);
    std::vector<int32_t> best_tag(m.N, INT32_MAX);
    for (int32_t f = 0; f < m.F; ++f) {
        const int32_t k = out.facet_kind[f];
        if (k >= 0) continue;
        for (int a = 0; a < 3; ++a) {
            const int32_t n = m.facets[3 * (size_t)f + a];
            if (m.facet_tag[f] < best_tag[n]) {
                best_tag[n] = m.facet_tag[f];
                out.dir_of_node[n] = -1 - k;
            }
        }
    }
    // initial_temperatures (+ index-keyed override)
    out.T0.resize(m.N);
#pragma omp parallel for schedule(static)
    for (int32_t n = 0; n < m.N; ++n) {
        out.T0[n] = s->initial_T ? s->initial_T[n] : s->materials[m.node_region[n]].initial_temperature;
        if (out.dir_of_node[n] >= 0) out.T0[n] = pl_eval(P, P.dir_tab[out.dir_of_node[n]], 0.0);
    }
    }
    // static dt (blocked.hpp:340-350): min_e rho c(0) l^2 / k(0). For constant
    // properties the bound is monotone in the element's minimum edge (also
    // under rounding), so the per-region minimum edge gives the exact minimum.
    if (!P.temp_dep) {
        double dt = INFINITY;
        for (int32_t r = 0; r < (int32_t)m.region_min_edge.size(); ++r) {
            if (!std::isfinite(m.region_min_edge[r])) continue;
            const DevMaterial& mm = P.mat[r];
            const double me = m.region_min_edge[r];
            dt = std::min(dt, mm.rho * mm.c0 * me * me / mm.k0);
        }
        out.min_bound = dt;
        P.static_dt = dt * s->dt_safety;
        if (!(P.static_dt > 0)) raise(CF_VALIDATION, "non-positive stable time step");
    }
}

// ------------------------------------------------------------------ tiles
void tile_env(TileCtx& c) {
    const char* so = std::getenv("CF_SLOT_ORDER");
    const char* sb = std::getenv("CF_SLOT_BANKS");
    c.slot_by_node = !(so && std::string(so) == "count");
    c.slot_banks = !(so && std::string(so) != "node") && !(sb && std::atoi(sb) == 0);
    const char* bp = std::getenv("CF_BANK_PASSES");
    c.bank_passes = bp ? std::atoi(bp) : 0;
    const char* bi = std::getenv("CF_BANK_ITERS");
    c.bank_iters = bi ? std::atoi(bi) : 0;
}

namespace {
inline uint64_t spread21(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

// Bank-aware local element positions (BankPlan, cf_tilepack.hpp). The tile kernel reads shared
// memory in two gathers:
//   phase 3: thread s (slot s) reads its j-th (lump, rc) operand pair, 16 B at pair index
//            q*S + pos(e) (S = ne2, a multiple of 8), so its 16-byte bank group is pos(e) & 7;
//   phase 2a: thread p (element at position p) reads sTH[slot of corner q], bank group slot & 7.
// An 8-thread quarter warp costs one shared-memory wavefront per distinct address in its most
// loaded bank group. The element positions are a free permutation (the reduction order is fixed
// by the CSR lists, ascending global element id): a greedy balanced colouring of the elements
// (colour = position & 7) spreads each phase-3 group over the bank groups, and optional in-block
// swaps (CF_BANK_PASSES) or a seeded local search (CF_BANK_ITERS) lower the wavefronts further.
// Deterministic: the same tile always yields the same positions.

// per-tile context of the shared tile functions (cf_tilepack.hpp) over the host arrays
TileCtx tile_ctx(const MeshData& m, const SetupData& S, const PlanOptions& o, const std::vector<int32_t>& fe_off,
                 const std::vector<int32_t>& fe, const std::vector<int32_t>& facet_sister, const uint8_t* kind_if) {
    TileCtx c;
    c.tets = m.tets.data();
    c.region = m.region;
    c.facets = m.facets;
    c.coords = m.coords;
    c.fe_off = fe_off.data();
    c.fe = fe.data();
    c.facet_kind = S.facet_kind.data();
    c.facet_sister = facet_sister.data();
    c.kind_interface = kind_if;
    c.tdep = S.temp_dep;
    c.coords_layout = o.geometry == CF_GEOM_COORDS;
    tile_env(c);
    return c;
}
}  // namespace

void build_rank_plan(const MeshData& m, const SetupData& S, const PlanOptions& o,
                     const std::vector<int32_t>& node_label, int32_t rank, RankPlan& rp) {
    rp = RankPlan{};
    rp.rank = rank;
    rp.coords = o.geometry == CF_GEOM_COORDS;
    const bool coords = rp.coords;
    const int32_t W = o.world_size;
    auto part_of = [&](int32_t e) { return W > 1 ? o.part_of_element[e] : 0; };

    // elements of this rank, ascending global id (SubDomain::from_elements blocked.hpp:25-39)
    std::vector<int32_t> elems;
    if (W == 1) {
        elems.resize(m.E);
#pragma omp parallel for schedule(static)
        for (int32_t e = 0; e < m.E; ++e) elems[e] = e;
    } else {  // ascending filter: per-thread counts, then fill
        const int nt = omp_get_max_threads();
        std::vector<int64_t> cnt(nt + 1, 0);
#pragma omp parallel num_threads(nt)
        {
            const int th = omp_get_thread_num();
            const int64_t lo = (int64_t)m.E * th / nt, hi = (int64_t)m.E * (th + 1) / nt;
            int64_t c = 0;
            for (int64_t e = lo; e < hi; ++e) c += part_of((int32_t)e) == rank;
            cnt[th + 1] = c;
#pragma omp barrier
#pragma omp single
            {
                for (int k = 0; k < nt; ++k) cnt[k + 1] += cnt[k];
                elems.resize(cnt[nt]);
            }
            int64_t j = cnt[th];
            for (int64_t e = lo; e < hi; ++e)
                if (part_of((int32_t)e) == rank) elems[j++] = (int32_t)e;
        }
    }
    const int64_t Er = (int64_t)elems.size();

    // parts touching each node (classify_nodes partition.hpp:311-327), only for W > 1
    std::vector<int64_t> np_off;
    std::vector<int32_t> np_parts;
    if (W > 1 && W <= 64) {
        // one bit per part, OR-ed in parallel; lists come out ascending
        std::vector<std::atomic<uint64_t>> mask(m.N);
#pragma omp parallel for schedule(static)
        for (int32_t n = 0; n < m.N; ++n) mask[n].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < (int64_t)m.E; ++e) {
            const uint64_t bit = 1ull << part_of((int32_t)e);
            for (int a = 0; a < 4; ++a) {
                std::atomic<uint64_t>& w = mask[m.tets[4 * (size_t)e + a]];
                if (!(w.load(std::memory_order_relaxed) & bit)) w.fetch_or(bit, std::memory_order_relaxed);
            }
        }
        np_off.assign(m.N + 1, 0);
        for (int32_t n = 0; n < m.N; ++n) np_off[n + 1] = np_off[n] + __builtin_popcountll(mask[n].load());
        np_parts.resize(np_off[m.N]);
#pragma omp parallel for schedule(static)
        for (int32_t n = 0; n < m.N; ++n) {
            uint64_t b = mask[n].load(std::memory_order_relaxed);
            int64_t j = np_off[n];
            while (b) {
                np_parts[j++] = __builtin_ctzll(b);
                b &= b - 1;
            }
        }
    } else if (W > 1) {
        np_off.assign(m.N + 1, 0);
        std::vector<int32_t> cnt(m.N, 0);
        std::vector<int64_t> off(m.N + 1, 0);
        for (int64_t i = 0; i < 4 * (int64_t)m.E; ++i) off[m.tets[i] + 1]++;
        for (int32_t n = 0; n < m.N; ++n) off[n + 1] += off[n];
        std::vector<int32_t> buf(off[m.N]);
        {
            std::vector<int64_t> cur(off.begin(), off.end() - 1);
            for (int64_t i = 0; i < 4 * (int64_t)m.E; ++i) buf[cur[m.tets[i]]++] = part_of((int32_t)(i / 4));
        }
        for (int32_t n = 0; n < m.N; ++n) {
            std::sort(buf.begin() + off[n], buf.begin() + off[n + 1]);
            cnt[n] = (int32_t)(std::unique(buf.begin() + off[n], buf.begin() + off[n + 1]) - (buf.begin() + off[n]));
            np_off[n + 1] = np_off[n] + cnt[n];
        }
        np_parts.resize(np_off[m.N]);
        for (int32_t n = 0; n < m.N; ++n)
            std::copy(buf.begin() + off[n], buf.begin() + off[n] + cnt[n], np_parts.begin() + np_off[n]);
    }
    trace_stage("plan: node parts");
    auto node_on = [&](int32_t n, int32_t p) {
        if (W == 1) return true;
        for (int64_t j = np_off[n]; j < np_off[n + 1]; ++j)
            if (np_parts[j] == p) return true;
        return false;
    };

    // facets per element (ascending facet id), Dirichlet facets excluded from bindings
    std::vector<char> in_rank(m.E, W == 1 ? 1 : 0);
    if (W > 1)
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < Er; ++i) in_rank[elems[i]] = 1;
    std::vector<int32_t> fe_off(m.E + 1, 0), fe;
    for (int32_t f = 0; f < m.F; ++f)
        if (in_rank[m.owner[f]] && S.facet_kind[f] >= 0) fe_off[m.owner[f] + 1]++;
    {  // parallel inclusive prefix sum over E + 1 entries (per-thread blocks, then offsets)
        const int nt = omp_get_max_threads();
        std::vector<int64_t> part(nt + 1, 0);
        const int64_t n1 = (int64_t)m.E + 1;
#pragma omp parallel num_threads(nt)
        {
            const int th = omp_get_thread_num();
            const int64_t lo = n1 * th / nt, hi = n1 * (th + 1) / nt;
            int64_t acc = 0;
            for (int64_t i = lo; i < hi; ++i) acc += fe_off[i];
            part[th + 1] = acc;
#pragma omp barrier
#pragma omp single
            for (int k = 0; k < nt; ++k) part[k + 1] += part[k];
            int64_t run = part[th];
            for (int64_t i = lo; i < hi; ++i) {
                run += fe_off[i];
                fe_off[i] = (int32_t)run;
            }
        }
    }
    fe.resize(fe_off[m.E]);
    {
        std::vector<int32_t> cur(fe_off.begin(), fe_off.end() - 1);
        for (int32_t f = 0; f < m.F; ++f)
            if (in_rank[m.owner[f]] && S.facet_kind[f] >= 0) fe[cur[m.owner[f]]++] = f;
    }

    std::vector<int32_t> facet_sister(m.F, -1);  // sister element of each interface facet
    for (size_t q = 0; q < S.pairs.size(); ++q) facet_sister[S.pairs[q].facet] = S.pairs[q].sister;
    uint8_t kind_if[kMaxFacetKinds];
    for (int k = 0; k < kMaxFacetKinds; ++k) kind_if[k] = (uint8_t)(S.P.kind[k].interface != 0);
    const TileCtx fc = tile_ctx(m, S, o, fe_off, fe, facet_sister, kind_if);
    trace_stage("plan: facet bindings");
    // ---- tiles: element order key, contiguous chunks, ascending id within a tile
    std::vector<std::vector<int32_t>> tiles;
    if (o.tile_of_element) {
        std::map<int32_t, std::vector<int32_t>> by;
        for (int32_t e : elems) by[o.tile_of_element[e]].push_back(e);
        for (auto& kv : by) tiles.push_back(std::move(kv.second));
    } else {
        std::vector<int32_t> order = elems;
        if (o.elem_order == CF_ELEM_ORDER_MORTON) {
            double lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY;
#pragma omp parallel for schedule(static) reduction(min : lo0, lo1, lo2) reduction(max : hi0, hi1, hi2)
            for (int32_t n = 0; n < m.N; ++n) {
                const double* q = m.pos(n);
                lo0 = std::min(lo0, q[0]);
                lo1 = std::min(lo1, q[1]);
                lo2 = std::min(lo2, q[2]);
                hi0 = std::max(hi0, q[0]);
                hi1 = std::max(hi1, q[1]);
                hi2 = std::max(hi2, q[2]);
            }
            const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
            const double span = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], 1e-300});
            struct Key {  // POD: the array is first touched by the parallel fill
                uint64_t code;
                int32_t e;
                bool operator<(const Key& b) const { return code != b.code ? code < b.code : e < b.e; }
            };
            std::vector<Key, UninitAlloc<Key>> key(Er);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < Er; ++i) {
                const int32_t e = elems[i];
                const int32_t* t = &m.tets[4 * (size_t)e];
                uint64_t code = 0;
                for (int k = 0; k < 3; ++k) {
                    const double c = 0.25 * (m.pos(t[0])[k] + m.pos(t[1])[k] + m.pos(t[2])[k] + m.pos(t[3])[k]);
                    double q = (c - lo[k]) / span * 2097151.0;
                    q = std::min(std::max(q, 0.0), 2097151.0);
                    code |= spread21((uint64_t)q) << k;
                }
                key[i] = Key{code, e};
            }
            trace_stage("plan: morton keys");
            __gnu_parallel::sort(key.begin(), key.end());  // keys unique: any sort gives this order
            trace_stage("plan: morton sort");
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < Er; ++i) order[i] = key[i].e;
        } else if (o.elem_order == CF_ELEM_ORDER_MIN_NODE) {
            std::vector<std::pair<int32_t, int32_t>> key(Er);
            for (int64_t i = 0; i < Er; ++i) {
                const int32_t e = elems[i];
                int32_t mn = INT32_MAX;
                for (int a = 0; a < 4; ++a) mn = std::min(mn, node_label[m.tets[4 * (size_t)e + a]]);
                key[i] = {mn, e};
            }
            std::sort(key.begin(), key.end());
            for (int64_t i = 0; i < Er; ++i) order[i] = key[i].second;
        }
        const int TE = o.tile_elems;
        for (int64_t i = 0; i < Er; i += TE)
            tiles.emplace_back(order.begin() + i, order.begin() + std::min<int64_t>(Er, i + TE));
        trace_stage("plan: chunks");
        // shared-memory budget: the 95th percentile of the chunk footprints; larger chunks
        // (interface / boundary chunks with many facets) are halved along the order until they
        // fit, so one launch configuration (and its occupancy) serves every tile
            auto footprint = [&](const int32_t* e0, int64_t n, std::vector<int32_t>& tab) {
            if (tab.size() < (size_t)(8 * n + 64)) tab.resize(8 * n + 64);
            return tile_footprint(fc, e0, (int)n, tab.data());
        };
        if (tiles.size() > 20) {
            std::vector<int64_t> fp(tiles.size());
#pragma omp parallel
            {
                std::vector<int32_t> tab;
#pragma omp for schedule(dynamic, 256)
                for (int64_t t = 0; t < (int64_t)tiles.size(); ++t)
                    fp[t] = footprint(tiles[t].data(), tiles[t].size(), tab);
            }
            std::vector<int64_t> srt = fp;
            const size_t q = (size_t)(0.95 * (double)(srt.size() - 1));
            std::nth_element(srt.begin(), srt.begin() + q, srt.end());
            int64_t budget = srt[q];
            // CF_SMEM_BUDGET=bytes caps it (e.g. so that 5 CTAs fit an SM's shared memory)
            if (const char* e = std::getenv("CF_SMEM_BUDGET")) budget = std::min<int64_t>(budget, std::atoll(e));
            std::vector<std::vector<int32_t>> out;
            out.reserve(tiles.size() + tiles.size() / 16);
            std::vector<std::vector<int32_t>> stack;
            std::vector<int32_t> tab;
            for (size_t t = 0; t < tiles.size(); ++t) {
                if (fp[t] <= budget) {
                    out.push_back(std::move(tiles[t]));
                    continue;
                }
                stack.assign(1, std::move(tiles[t]));
                while (!stack.empty()) {  // depth-first halves keep the order
                    std::vector<int32_t> c = std::move(stack.back());
                    stack.pop_back();
                    if (c.size() <= 16 || footprint(c.data(), c.size(), tab) <= budget) {
                        out.push_back(std::move(c));
                        continue;
                    }
                    const size_t h = c.size() / 2;
                    stack.emplace_back(c.begin() + h, c.end());
                    stack.emplace_back(c.begin(), c.begin() + h);
                }
            }
            tiles.swap(out);
        }
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t t = 0; t < (int64_t)tiles.size(); ++t) std::sort(tiles[t].begin(), tiles[t].end());
    trace_stage("plan: tiles");
    for (auto& t : tiles)
        if ((int)t.size() > kMaxTileElems)
            raise(CF_INVALID_ARG, "a tile holds more than 2048 elements (" + std::to_string(t.size()) + ")");

    // ---- local node numbering: given / RCM label / first touch in tile order
    std::vector<int32_t> local_of(m.N, -1);
    std::vector<int32_t> lnodes;
    if (o.node_order == CF_NODE_ORDER_TILE) {
        // first touch in tile order, in parallel: each thread owns a contiguous range of
        // tiles; a node belongs to the first range touching it (atomic min of the range
        // index), the owner lists its nodes in first-touch order, lists concatenate in
        // range order -- the serial first-touch order exactly
        const int nt = omp_get_max_threads();
        const int64_t T_ = (int64_t)tiles.size();
        std::vector<std::atomic<int32_t>> owner(m.N);
        std::vector<std::vector<int32_t>> lists(nt);
#pragma omp parallel num_threads(nt)
        {
            const int th = omp_get_thread_num();
#pragma omp for schedule(static)
            for (int32_t n = 0; n < m.N; ++n) owner[n].store(INT32_MAX, std::memory_order_relaxed);
            const int64_t lo = T_ * th / nt, hi = T_ * (th + 1) / nt;
            for (int64_t t = lo; t < hi; ++t)
                for (int32_t e : tiles[t])
                    for (int a = 0; a < 4; ++a) {
                        std::atomic<int32_t>& w = owner[m.tets[4 * (size_t)e + a]];
                        int32_t cur = w.load(std::memory_order_relaxed);
                        while (th < cur && !w.compare_exchange_weak(cur, th, std::memory_order_relaxed)) {
                        }
                    }
#pragma omp barrier
            auto& L = lists[th];
            std::vector<uint64_t> seen(((size_t)m.N + 63) / 64, 0);  // private: no shared-line writes
            for (int64_t t = lo; t < hi; ++t)
                for (int32_t e : tiles[t])
                    for (int a = 0; a < 4; ++a) {
                        const int32_t n = m.tets[4 * (size_t)e + a];
                        const uint64_t bit = 1ull << (n & 63);
                        if (!(seen[n >> 6] & bit) && owner[n].load(std::memory_order_relaxed) == th) {
                            seen[n >> 6] |= bit;
                            L.push_back(n);
                        }
                    }
        }
        std::vector<int64_t> off(nt + 1, 0);
        for (int k = 0; k < nt; ++k) off[k + 1] = off[k] + (int64_t)lists[k].size();
        lnodes.resize(off[nt]);
#pragma omp parallel for schedule(static, 1)
        for (int k = 0; k < nt; ++k)
            for (size_t i = 0; i < lists[k].size(); ++i) {
                lnodes[off[k] + i] = lists[k][i];
                local_of[lists[k][i]] = (int32_t)(off[k] + i);
            }
    } else {
        std::vector<char> mark(m.N, 0);
        for (int32_t e : elems)
            for (int a = 0; a < 4; ++a) mark[m.tets[4 * (size_t)e + a]] = 1;
        for (int32_t n = 0; n < m.N; ++n)
            if (mark[n]) lnodes.push_back(n);
        if (o.node_order == CF_NODE_ORDER_RCM)
            std::sort(lnodes.begin(), lnodes.end(),
                      [&](int32_t a, int32_t b) { return node_label[a] < node_label[b]; });
        for (size_t i = 0; i < lnodes.size(); ++i) local_of[lnodes[i]] = (int32_t)i;
    }
    trace_stage("plan: local numbering");
    rp.n_local = (int32_t)lnodes.size();
    if (rp.n_local >= (1 << 28)) raise(CF_INVALID_ARG, "more than 2^28 nodes on one rank");

    // ghosts: sister nodes of this rank's interface facets that are not local
    std::vector<int32_t> ghosts;
    for (int32_t f = 0; f < m.F; ++f) {
        if (!in_rank[m.owner[f]] || S.facet_kind[f] < 0 || !S.P.kind[S.facet_kind[f]].interface) continue;
        const int32_t sis = S.pairs[S.pair_of_facet[f]].sister;
        for (int a = 0; a < 4; ++a) {
            const int32_t n = m.tets[4 * (size_t)sis + a];
            if (local_of[n] < 0) ghosts.push_back(n);
        }
    }
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    rp.n_ghost = (int32_t)ghosts.size();
    for (size_t g = 0; g < ghosts.size(); ++g) local_of[ghosts[g]] = rp.n_local + (int32_t)g;
    rp.local_global = lnodes;
    rp.local_global.insert(rp.local_global.end(), ghosts.begin(), ghosts.end());

    trace_stage("plan: ghosts");
    rp.node_region.resize(rp.n_local);
    for (int32_t l = 0; l < rp.n_local; ++l) rp.node_region[l] = (uint8_t)m.node_region[lnodes[l]];
    bool any_dir = false;
    for (int32_t l = 0; l < rp.n_local; ++l)
        if (S.dir_of_node[lnodes[l]] >= 0) any_dir = true;
    if (any_dir) {
        rp.node_dir.resize(rp.n_local);
        for (int32_t l = 0; l < rp.n_local; ++l) rp.node_dir[l] = (int8_t)S.dir_of_node[lnodes[l]];
    }

    // ---- per tile: slots, CSR, facet bindings, packed into the blob.
    // Pass 1 (parallel): each tile's slot list and sizes; tiles over the shared-memory
    // budget are halved along the element order (their slot lists recomputed); sizes ->
    // offsets; pass 2 (parallel): fill the tile's blob section at its offset.
    const int nthr = omp_get_max_threads();
    std::vector<std::vector<int32_t>> tile_nodes;
    std::vector<TileMeta> meta;
    TileCtx tc = fc;
    tc.local_of = local_of.data();
    auto pass1 = [&](const std::vector<int32_t>& which) {
#pragma omp parallel num_threads(nthr)
        {
            std::vector<int32_t> ws, tmp;
#pragma omp for schedule(dynamic, 64)
            for (int64_t w = 0; w < (int64_t)which.size(); ++w) {
                const int32_t t = which[w];
                const auto& te = tiles[t];
                const size_t need = 8 * te.size() + 8 * 4 * te.size() + 64;
                if (ws.size() < need) ws.resize(need);
                if (tmp.size() < 4 * te.size()) tmp.resize(4 * te.size());
                meta[t] = tile_pass1(tc, te.data(), (int)te.size(), tmp.data(), ws.data());
                tile_nodes[t].assign(tmp.begin(), tmp.begin() + meta[t].ns);
            }
        }
    };
    tile_nodes.resize(tiles.size());
    meta.resize(tiles.size());
    {
        std::vector<int32_t> all(tiles.size());
        std::iota(all.begin(), all.end(), 0);
        pass1(all);
    }
    rp.n_tiles = (int32_t)tiles.size();
    rp.tile_meta = meta;
    trace_stage("plan: tile slots");

    // node -> number of tiles touching it (tile-private test), rank-shared nodes, border tiles
    std::vector<int32_t> ntiles_of(rp.n_local, 0);
#pragma omp parallel for schedule(dynamic, 256)
    for (int32_t t = 0; t < rp.n_tiles; ++t)
        for (int32_t l : tile_nodes[t]) std::atomic_ref<int32_t>(ntiles_of[l]).fetch_add(1, std::memory_order_relaxed);
    std::vector<char> shared_node(rp.n_local, 0);
    if (W > 1)
        for (int32_t l = 0; l < rp.n_local; ++l) {
            const int32_t n = lnodes[l];
            shared_node[l] = (np_off[n + 1] - np_off[n]) > 1;
        }
    rp.tile_border.assign(rp.n_tiles, 0);
    if (W > 1)
        for (int32_t t = 0; t < rp.n_tiles; ++t) {  // border tile: holds a rank-shared node
            bool b = false;
            for (int32_t l : tile_nodes[t]) b = b || shared_node[l];
            rp.tile_border[t] = b;
        }
    // slot order inside a tile (tile_pack): tile-private nodes first (by contribution count,
    // descending: similar reduction-list lengths share a warp), then the tile-shared nodes in
    // ascending node id, so the partials they write and the slot copies the update kernel writes
    // back are laid out in the update's (node) order -- whole sectors instead of scattered 16 /
    // 8-byte accesses
    rp.tile_slot_off.assign(rp.n_tiles + 1, 0);
    rp.blob_off.assign(rp.n_tiles + 1, 0);
    rp.elem_global.resize(Er);
    std::vector<int64_t> elem_off(rp.n_tiles + 1, 0);
    for (int32_t t = 0; t < rp.n_tiles; ++t) {  // no throwing inside the parallel regions
        const TileMeta& tm = rp.tile_meta[t];
        const TileLayout L(tm, S.temp_dep, coords);
        if (4 * tm.ne + 4 * tm.nf > 65535 || tm.ncsr > 65535 || tm.ne > 1024 || L.max_operand() > 0x7fff)
            raise(CF_INVALID_ARG, "tile too large for 16-bit slot / operand indices (at most 1024 tets per tile)");
    }
    for (int32_t t = 0; t < rp.n_tiles; ++t) {
        const TileMeta& tm = rp.tile_meta[t];
        const TileLayout L(tm, S.temp_dep, coords);
        rp.blob_off[t + 1] = rp.blob_off[t] + L.total;  // copied part + the stored layout's max_edge tail
        rp.tile_slot_off[t + 1] = rp.tile_slot_off[t] + (int32_t)cf_round(tm.ns, 2);  // 16 B aligned Tslot segments
        elem_off[t + 1] = elem_off[t] + tm.ne;
        rp.max_elems = std::max(rp.max_elems, tm.ne);
        rp.max_slots = std::max(rp.max_slots, (int32_t)cf_round(tm.ns, 2));
        rp.max_facets = std::max(rp.max_facets, tm.nf);
        rp.max_blob = std::max<int64_t>(rp.max_blob, L.bytes);
        rp.max_scratch = std::max<int64_t>(rp.max_scratch, L.scratch);
    }
    // host staging holds each tile's connectivity and non-geometry sections only
    // (TileLayout::staged_bytes); the geometry pairs (or slot coordinates) are computed on the
    // device from tets_ord / coords_local (fill_tiles_kernel, the host tet_geometry's operation
    // order), so the host never holds the 88 B/tet of ElementGeom.
    rp.rest_off.assign(rp.n_tiles + 1, 0);
    for (int32_t t = 0; t < rp.n_tiles; ++t)
        rp.rest_off[t + 1] = rp.rest_off[t] + TileLayout(rp.tile_meta[t], S.temp_dep, coords).staged_bytes();
    rp.blob_bytes = rp.blob_off[rp.n_tiles];
    rp.blob.resize(rp.rest_off[rp.n_tiles]);
    rp.elem_off.assign(elem_off.begin(), elem_off.end());
    rp.tets_ord.resize(4 * (size_t)Er);
    rp.coords_local.resize(3 * (size_t)rp.n_local);
#pragma omp parallel for schedule(static)
    for (int32_t l = 0; l < rp.n_local; ++l)
        for (int k = 0; k < 3; ++k) rp.coords_local[3 * (size_t)l + k] = m.pos(lnodes[l])[k];
    rp.slot_node.resize(rp.tile_slot_off[rp.n_tiles]);
    int64_t n_if = 0, n_bc = 0, bank_after = 0, bank_a = 0, bank_b = 0, bank_ib = 0;
    const bool bank_trace = std::getenv("CF_TRACE_SETUP") && std::atoi(std::getenv("CF_TRACE_SETUP"));
    tc.lnode_region = rp.node_region.data();
    tc.lnode_dir = rp.node_dir.empty() ? nullptr : rp.node_dir.data();
    tc.ntiles_of = ntiles_of.data();
    std::vector<uint8_t> shared_u8;
    if (W > 1) {
        shared_u8.assign(shared_node.begin(), shared_node.end());
        tc.shared_node = shared_u8.data();
    }
    TileCaps caps{1, 1, 0, 0};
    for (int32_t t = 0; t < rp.n_tiles; ++t) {
        const TileMeta& tm = rp.tile_meta[t];
        caps.ne = std::max(caps.ne, tm.ne);
        caps.ns = std::max(caps.ns, tm.ns);
        caps.nf = std::max(caps.nf, tm.nf);
        caps.ncsr = std::max(caps.ncsr, tm.ncsr);
    }
    const int64_t ws_ints = tile_ws_ints(caps);
#pragma omp parallel num_threads(nthr) reduction(+ : n_if, n_bc, bank_after, bank_a, bank_b, bank_ib)
    {
        std::vector<int32_t> ws(ws_ints);
#pragma omp for schedule(dynamic, 64)
        for (int32_t t = 0; t < rp.n_tiles; ++t) {
            const TileMeta tm = rp.tile_meta[t];
            const TileLayout L(tm, S.temp_dep, coords);
            uint8_t* const stg = rp.blob.data() + rp.rest_off[t];  // connectivity first, then sections >= stage
            std::memset(stg, 0, (size_t)L.staged_bytes());
            TileOut to;
            to.stg = stg;
            to.elem_global = rp.elem_global.data() + elem_off[t];
            to.tets_ord = rp.tets_ord.data() + 4 * elem_off[t];
            to.slot_node = rp.slot_node.data() + rp.tile_slot_off[t];
            tile_pack(tc, t, tiles[t].data(), tm, tile_nodes[t].data(), ws.data(), to, bank_trace);
            n_if += to.n_if;
            n_bc += to.n_bc;
            if (bank_trace && !coords && tm.ne >= 16) {
                bank_after += to.bank_cost[0];
                bank_a += to.bank_cost[1];
                bank_b += to.bank_cost[2];
                bank_ib += 4 * ((tm.ne + 7) / 8);
            }
        }
    }
    if (bank_trace)
        std::fprintf(stderr, "[cf setup] rank %d bank-aware positions: shared-memory wavefronts %lld "
                     "(reduction reads %lld; corner gathers %lld, ideal %lld)\n", rank,
                     (long long)bank_after, (long long)bank_a, (long long)bank_b, (long long)bank_ib);
    rp.n_if_facets = n_if;
    rp.n_bc_facets = n_bc;
    std::vector<std::vector<int32_t>>().swap(tile_nodes);
    trace_stage("plan: blob packing");
    // merge lists: ascending tile per node (merge_offsets/merge_entries blocked.hpp:294-307)
    const int64_t S_tot = rp.tile_slot_off[rp.n_tiles];
    rp.merge_off.assign(rp.n_local + 1, 0);
    auto snode = [&](int64_t s) { return (int32_t)((uint32_t)rp.slot_node[s] & 0x0fffffffu); };
    for (int64_t s = 0; s < S_tot; ++s)
        if (rp.slot_node[s] >= 0) rp.merge_off[snode(s) + 1]++;
    for (int32_t l = 0; l < rp.n_local; ++l) rp.merge_off[l + 1] += rp.merge_off[l];
    rp.merge_idx.resize(S_tot);
    {
        std::vector<int32_t> cur(rp.merge_off.begin(), rp.merge_off.end() - 1);
        for (int64_t s = 0; s < S_tot; ++s)
            if (rp.slot_node[s] >= 0) rp.merge_idx[cur[snode(s)]++] = (int32_t)s;
    }
    for (int32_t l = 0; l < rp.n_local; ++l) {
        if (ntiles_of[l] == 1 && !shared_node[l]) rp.n_private++;
        else rp.shared_list.push_back(l);
    }
    // the update kernel walks its nodes in the order of their first partial (the tile order), so
    // consecutive threads read neighbouring partials and write neighbouring slot copies whatever
    // the node numbering (RCM labels sweep a front across the mesh; first-touch numbering already
    // follows the tiles, for which this order is the node order)
    {
        std::vector<std::pair<int64_t, int32_t>> key(rp.shared_list.size());  // first partials are unique
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < (int64_t)key.size(); ++k) {
            const int32_t l = rp.shared_list[k];
            key[k] = {rp.merge_off[l + 1] > rp.merge_off[l] ? (int64_t)rp.merge_idx[rp.merge_off[l]]
                                                             : INT64_MAX - rp.n_local + l,
                      l};
        }
        __gnu_parallel::sort(key.begin(), key.end());
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < (int64_t)key.size(); ++k) rp.shared_list[k] = key[k].second;
    }

    trace_stage("plan: merge lists");
    // ---------------------------------------------------- multi-rank exchange
    if (W > 1) {
        // need(p, q) = nodes part p needs from part q (external_from partition.hpp:346-354)
        auto ext_need = [&](int32_t p, int32_t q) {
            std::vector<int32_t> v;
            for (int32_t f = 0; f < m.F; ++f) {
                if (part_of(m.owner[f]) != p || S.facet_kind[f] < 0 || !S.P.kind[S.facet_kind[f]].interface) continue;
                const int32_t sis = S.pairs[S.pair_of_facet[f]].sister;
                if (part_of(sis) != q) continue;
                for (int a = 0; a < 4; ++a) {
                    const int32_t n = m.tets[4 * (size_t)sis + a];
                    if (!node_on(n, p)) v.push_back(n);
                }
            }
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            return v;
        };
        std::map<int32_t, RankPlan::Neighbor> nb;
        std::vector<int32_t> shared;  // ascending global id
        for (int32_t l = 0; l < rp.n_local; ++l)
            if (shared_node[l]) shared.push_back(lnodes[l]);
        std::sort(shared.begin(), shared.end());
        rp.n_shared = (int64_t)shared.size();
        rp.node_shared.assign(rp.n_local, -1);
        for (size_t i = 0; i < shared.size(); ++i) rp.node_shared[local_of[shared[i]]] = (int32_t)i;
        for (int32_t n : shared)
            for (int64_t j = np_off[n]; j < np_off[n + 1]; ++j)
                if (np_parts[j] != rank) nb[np_parts[j]].shared.push_back(local_of[n]);
        for (int32_t q = 0; q < W; ++q) {
            if (q == rank) continue;
            auto from = ext_need(rank, q);
            auto to = ext_need(q, rank);
            if (from.empty() && to.empty() && !nb.count(q)) continue;
            auto& x = nb[q];
            for (int32_t n : from) x.ext_from.push_back(local_of[n]);
            for (int32_t n : to) {
                if (local_of[n] < 0 || local_of[n] >= rp.n_local) raise(CF_PROTOCOL, "external node not local to sender");
                x.ext_to.push_back(local_of[n]);
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
        // combine lists per shared node: ascending rank, own = -1
        std::vector<std::vector<std::array<int32_t, 3>>> src(shared.size());
        for (size_t i = 0; i < shared.size(); ++i) src[i].push_back({rank, -1, -1});
        for (size_t k = 0; k < rp.nbrs.size(); ++k) {
            const auto& x = rp.nbrs[k];
            const int32_t ns = (int32_t)x.shared.size();
            for (int32_t j = 0; j < ns; ++j)
                src[rp.node_shared[x.shared[j]]].push_back(
                    {x.rank, (int32_t)(rp.recv_off[k] + j), (int32_t)(rp.recv_off[k] + ns + j)});
        }
        rp.shared_off.assign(shared.size() + 1, 0);
        for (size_t i = 0; i < shared.size(); ++i) {
            std::sort(src[i].begin(), src[i].end());
            rp.shared_off[i + 1] = rp.shared_off[i] + (int32_t)src[i].size();
            for (auto& pr : src[i]) {
                rp.shared_src.push_back(pr[1]);
                rp.shared_src_r.push_back(pr[2]);
            }
        }
        // ghost sources: first neighbour (ascending rank) providing the node
        rp.ghost_src.assign(rp.n_ghost, -1);
        for (size_t k = 0; k < rp.nbrs.size(); ++k) {
            const auto& x = rp.nbrs[k];
            const int64_t base = rp.recv_off[k] + 2 * (int64_t)x.shared.size();
            for (size_t j = 0; j < x.ext_from.size(); ++j) {
                const int32_t g = x.ext_from[j] - rp.n_local;
                if (g >= 0 && rp.ghost_src[g] < 0) rp.ghost_src[g] = (int32_t)(base + (int64_t)j);
            }
        }
        for (int32_t g = 0; g < rp.n_ghost; ++g)
            if (rp.ghost_src[g] < 0) raise(CF_PROTOCOL, "ghost node without a provider");
        trace_stage("plan: exchange lists");
    }
}

}  // namespace cfb
