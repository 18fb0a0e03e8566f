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
    for (int32_t e = 0; e < m.E; ++e)
        if (m.region[e] >= s->n_materials)
            raise(CF_CONFIG, "no material for region " + std::to_string(m.region[e]));
    if (s->n_materials > kMaxRegions) raise(CF_CONFIG, "more than 16 material regions");
    std::vector<char> used(s->n_materials + 1, 0);
    for (int32_t r = 0; r < m.region_count; ++r) used[r] = 0;
    for (int32_t e = 0; e < m.E; ++e) used[m.region[e]] = 1;
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
    out.facet_kind.resize(m.F);
    for (int32_t f = 0; f < m.F; ++f) {
        out.facet_kind[f] = kind_of_tag[m.facet_tag[f]];
        if (out.facet_kind[f] >= 0 && P.kind[out.facet_kind[f]].interface && out.pair_of_facet[f] < 0)
            raise(CF_CONFIG, "interface facet " + std::to_string(f) + " has no sister pairing; call pair_sister_facets");
    }
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

// Bank-aware local element positions. The tile kernel reads shared memory in two gathers:
//   phase 3: thread s (slot s) reads its j-th (lump, rc) operand pair, 16 B at pair index
//            q*S + pos(e) (S = ne2, a multiple of 8), so its 16-byte bank group is pos(e) & 7;
//   phase 2a: thread p (element at position p) reads sTH[slot of corner q], bank group slot & 7.
// An 8-thread quarter warp costs one shared-memory wavefront per distinct address in its most
// loaded bank group. The element positions are a free permutation (the reduction order is fixed
// by the CSR lists, ascending global element id): a greedy balanced colouring of the elements
// (colour = position & 7) spreads each phase-3 group over the bank groups (cfg2: 1.63x -> ~1.3x
// the ideal wavefronts of random positions... see DESIGN.md), and an optional seeded local search
// over position swaps (CF_BANK_ITERS) lowers the summed wavefronts of both gathers further.
// `items` are the slots' operand lists in reduction
// order, padded like the CSR: element corner (i << 2 | q) or 0x80000000 | fixed pair address.
// Deterministic: the same tile always yields the same positions.
struct BankPlanner {
    int ne, ns;
    std::vector<int32_t> pos, at;            // element -> position, position -> element
    std::vector<int32_t> a_off, a_items;     // phase-3 groups (quarter warp of slots, list index)
    std::vector<int32_t> g_off, g_list;      // element -> its phase-3 groups
    const int32_t* eslot = nullptr;          // element i, corner q -> slot
    int cost_a(int g) const {
        int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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
                cnt[ad & 7]++;
            } else {
                cnt[pos[it >> 2] & 7]++;
            }
        }
        int mx = 0;
        for (int b = 0; b < 8; ++b) mx = std::max(mx, cnt[b]);
        return mx;
    }
    int cost_b(int blk, int q) const {  // quarter warp of element positions, corner q
        int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int32_t seen[8];
        int ns_ = 0;
        for (int p = 8 * blk; p < std::min(ne, 8 * blk + 8); ++p) {
            const int32_t sl = eslot[4 * at[p] + q];
            bool dup = false;
            for (int k = 0; k < ns_; ++k) dup = dup || seen[k] == sl;
            if (dup) continue;
            seen[ns_++] = sl;
            cnt[sl & 7]++;
        }
        int mx = 0;
        for (int b = 0; b < 8; ++b) mx = std::max(mx, cnt[b]);
        return mx;
    }
    // items: per slot [off[s], off[s+1]) in reduction order (already padded to multiples of 4)
    const int32_t* sperm = nullptr;          // phase-3 thread j reduces slot sperm[j] (null: j)
    void run(int ne_, int ns_, const int32_t* eslot_, const std::vector<int32_t>& off,
             const std::vector<uint32_t>& items, int iters, uint64_t seed, bool greedy = true) {
        ne = ne_;
        ns = ns_;
        eslot = eslot_;
        pos.resize(ne);
        at.resize(ne);
        std::iota(pos.begin(), pos.end(), 0);
        std::iota(at.begin(), at.end(), 0);
        if (ne < 16) return;
        // phase-3 groups
        a_off.assign(1, 0);
        a_items.clear();
        auto slot_at = [&](int j) { return sperm ? sperm[j] : j; };
        for (int q0 = 0; q0 < ns; q0 += 8) {
            int mx = 0;
            for (int u = q0; u < std::min(ns, q0 + 8); ++u) mx = std::max(mx, off[slot_at(u) + 1] - off[slot_at(u)]);
            for (int j = 0; j < mx; ++j) {
                for (int u = q0; u < std::min(ns, q0 + 8); ++u) {
                    const int sl = slot_at(u);
                    if (off[sl] + j < off[sl + 1]) a_items.push_back((int32_t)items[off[sl] + j]);
                }
                a_off.push_back((int32_t)a_items.size());
            }
        }
        const int na = (int)a_off.size() - 1;
        g_off.assign(ne + 1, 0);
        for (int g = 0; g < na; ++g)
            for (int k = a_off[g]; k < a_off[g + 1]; ++k)
                if (!((uint32_t)a_items[k] & 0x80000000u)) g_off[((uint32_t)a_items[k] >> 2) + 1]++;
        for (int i = 0; i < ne; ++i) g_off[i + 1] += g_off[i];
        g_list.resize(g_off[ne]);
        {
            std::vector<int32_t> cur(g_off.begin(), g_off.end() - 1);
            for (int g = 0; g < na; ++g)
                for (int k = a_off[g]; k < a_off[g + 1]; ++k)
                    if (!((uint32_t)a_items[k] & 0x80000000u)) g_list[cur[(uint32_t)a_items[k] >> 2]++] = g;
        }
        // greedy balanced colouring: each element takes the bank group (position & 7) least used by
        // the other members of its phase-3 groups, within the group's capacity (positions < ne)
        if (greedy) {
            std::vector<int32_t> cnt(8 * (size_t)na, 0);
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
                    cnt[8 * (size_t)g + (ad & 7)]++;
                }
            }
            // blocks of 8 consecutive elements (reference order: spatially coherent, so the
            // phase-2a corner gathers keep their broadcasts) take the 8 colours as a permutation
            for (int b0 = 0; b0 < ne; b0 += 8) {
                const int nb = std::min(8, ne - b0);
                bool used[8] = {false, false, false, false, false, false, false, false};
                for (int i = b0; i < b0 + nb; ++i) {
                    int best = -1, best_score = 1 << 30;
                    for (int c = 0; c < nb; ++c) {  // a partial last block uses positions b0 .. ne-1
                        if (used[c]) continue;
                        // score: added wavefronts (a count reaching its group's maximum), then load
                        int sc = 0;
                        for (int k = g_off[i]; k < g_off[i + 1]; ++k) {
                            const int32_t* cg = &cnt[8 * (size_t)g_list[k]];
                            int mx = 0;
                            for (int u = 0; u < 8; ++u) mx = std::max(mx, cg[u]);
                            sc += 64 * (cg[c] + 1 > mx) + cg[c];
                        }
                        if (sc < best_score) {
                            best_score = sc;
                            best = c;
                        }
                    }
                    used[best] = true;
                    for (int k = g_off[i]; k < g_off[i + 1]; ++k) cnt[8 * (size_t)g_list[k] + best]++;
                    pos[i] = b0 + best;
                    at[b0 + best] = i;
                }
            }
            // refinement (CF_BANK_PASSES, default 0): pairwise colour swaps inside a block (the
            // block's corner gathers are unchanged) while they lower the reduction-read wavefronts.
            // cfg2: 3 passes take the reduction reads from 1.80x to 1.67x the ideal for -0.5 % tile
            // time, but cost ~2 s of setup per 12.6 M tets (cfg5: ~30 s), so they are opt-in.
            const char* rp_env = std::getenv("CF_BANK_PASSES");
            const int refine_passes = rp_env ? std::atoi(rp_env) : 0;
            auto gmax = [&](int g) {
                const int32_t* cg = &cnt[8 * (size_t)g];
                int mx = 0;
                for (int u = 0; u < 8; ++u) mx = std::max(mx, cg[u]);
                return mx;
            };
            int touched[16];
            for (int pass = 0; pass < refine_passes; ++pass) {
                bool improved = false;
                for (int b0 = 0; b0 < ne; b0 += 8) {
                    const int nb = std::min(8, ne - b0);
                    for (int u = 0; u < nb; ++u)
                        for (int v = u + 1; v < nb; ++v) {
                            const int i1 = at[b0 + u], i2 = at[b0 + v];
                            const int c1 = pos[i1] & 7, c2 = pos[i2] & 7;
                            int nt = 0;
                            for (int i : {i1, i2})
                                for (int k = g_off[i]; k < g_off[i + 1]; ++k) {
                                    bool dup = false;
                                    for (int w = 0; w < nt; ++w) dup = dup || touched[w] == g_list[k];
                                    if (!dup && nt < 16) touched[nt++] = g_list[k];
                                }
                            int before = 0;
                            for (int w = 0; w < nt; ++w) before += gmax(touched[w]);
                            auto move = [&](int i, int from, int to) {
                                for (int k = g_off[i]; k < g_off[i + 1]; ++k) {
                                    cnt[8 * (size_t)g_list[k] + from]--;
                                    cnt[8 * (size_t)g_list[k] + to]++;
                                }
                            };
                            move(i1, c1, c2);
                            move(i2, c2, c1);
                            int after = 0;
                            for (int w = 0; w < nt; ++w) after += gmax(touched[w]);
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
        auto rnd = [&]() {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            return x;
        };
        int ga[16], gb[4];
        for (int it = 0; it < iters; ++it) {
            const int i1 = (int)(rnd() % (uint64_t)ne), i2 = (int)(rnd() % (uint64_t)ne);
            const int p1 = pos[i1], p2 = pos[i2];
            if ((p1 & 7) == (p2 & 7) && (p1 >> 3) == (p2 >> 3)) continue;
            int na_ = 0;
            for (int i : {i1, i2})
                for (int k = g_off[i]; k < g_off[i + 1]; ++k) {
                    bool dup = false;
                    for (int u = 0; u < na_; ++u) dup = dup || ga[u] == g_list[k];
                    if (!dup && na_ < 16) ga[na_++] = g_list[k];
                }
            const int nb = (p1 >> 3) == (p2 >> 3) ? 1 : 2;
            gb[0] = p1 >> 3;
            gb[1] = p2 >> 3;
            auto total = [&]() {
                int c = 0;
                for (int u = 0; u < na_; ++u) c += cost_a(ga[u]);
                for (int u = 0; u < nb; ++u)
                    for (int q = 0; q < 4; ++q) c += cost_b(gb[u], q);
                return c;
            };
            const int before = total();
            std::swap(pos[i1], pos[i2]);
            at[p1] = i2;
            at[p2] = i1;
            if (total() > before) {  // revert (sideways moves are kept)
                std::swap(pos[i1], pos[i2]);
                at[p1] = i1;
                at[p2] = i2;
            }
        }
    }
    int total_cost(int which = 3) const {  // 1: phase-3 reads, 2: phase-2a gathers
        int c = 0;
        if (which & 1)
            for (int g = 0; g + 1 < (int)a_off.size(); ++g) c += cost_a(g);
        if (which & 2)
            for (int b = 0; 8 * b < ne; ++b)
                for (int q = 0; q < 4; ++q) c += cost_b(b, q);
        return c;
    }
    int n_groups(int which) const { return which == 1 ? (int)a_off.size() - 1 : 4 * ((ne + 7) / 8); }
};
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
        auto footprint = [&](const int32_t* e0, int64_t n, std::vector<int64_t>& tab) {
            // unique nodes and their contribution counts: open addressing on (node, count)
            size_t cap = 64;
            while (cap < 8 * (size_t)n) cap <<= 1;
            if (tab.size() < cap) tab.resize(cap);
            std::fill(tab.begin(), tab.begin() + cap, -1);
            const size_t mask = cap - 1;
            int ns = 0, nf = 0;
            auto add = [&](int32_t v) {
                size_t h = ((uint64_t)(uint32_t)v * 0x9E3779B97F4A7C15ull) >> 32 & mask;
                while (tab[h] >= 0 && (int32_t)(tab[h] >> 32) != v) h = (h + 1) & mask;
                if (tab[h] < 0) {
                    tab[h] = (int64_t)v << 32;
                    ++ns;
                }
                tab[h] += 1;
            };
            for (int64_t i = 0; i < n; ++i) {
                const int32_t e = e0[i];
                for (int a = 0; a < 4; ++a) add(m.tets[4 * (size_t)e + a]);
                for (int32_t j = fe_off[e]; j < fe_off[e + 1]; ++j, ++nf)
                    for (int a = 0; a < 3; ++a) add(m.facets[3 * (size_t)fe[j] + a]);
            }
            int ncsr = 0;
            for (size_t h = 0; h < cap; ++h)
                if (tab[h] >= 0) ncsr += ((int)(tab[h] & 0xffffffff) + 3) & ~3;
            const TileLayout L(TileMeta{(int32_t)n, ns, nf, ncsr}, S.temp_dep, o.geometry == CF_GEOM_COORDS);
            return (int64_t)cf_round(L.bytes, 16) + 24 * cf_round(ns, 2) + 8 * cf_round(L.scratch, 2);
        };
        if (tiles.size() > 20) {
            std::vector<int64_t> fp(tiles.size());
#pragma omp parallel
            {
                std::vector<int64_t> tab;
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
            std::vector<int64_t> tab;
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
    auto tile_facets = [&](const std::vector<int32_t>& te, std::vector<int32_t>& out) {
        out.clear();  // facet bindings, element order then facet id (blocked.hpp:244-288)
        for (int32_t e : te)
            for (int32_t j = fe_off[e]; j < fe_off[e + 1]; ++j) out.push_back(fe[j]);
    };
    auto pass1 = [&](const std::vector<int32_t>& which) {
#pragma omp parallel num_threads(nthr)
        {
            std::vector<int32_t> slot_of(rp.n_local, -1), cnt_of, idx, tfacets, sorted;
#pragma omp for schedule(dynamic, 64)
            for (int64_t w = 0; w < (int64_t)which.size(); ++w) {
                const int32_t t = which[w];
                const auto& te = tiles[t];
                auto& tnodes = tile_nodes[t];
                tnodes.clear();
                for (int32_t e : te)
                    for (int a = 0; a < 4; ++a) {
                        const int32_t l = local_of[m.tets[4 * (size_t)e + a]];
                        if (slot_of[l] == -1) {
                            slot_of[l] = -2;
                            tnodes.push_back(l);
                        }
                    }
                // slots ordered by contribution count (desc), then local id: the warps of
                // the reduction phase then walk lists of near-equal length (no divergence)
                for (size_t k = 0; k < tnodes.size(); ++k) slot_of[tnodes[k]] = (int32_t)k;
                cnt_of.assign(tnodes.size(), 0);
                tile_facets(te, tfacets);
                for (int32_t e : te)
                    for (int a = 0; a < 4; ++a) cnt_of[slot_of[local_of[m.tets[4 * (size_t)e + a]]]]++;
                for (int32_t f : tfacets)
                    for (int a = 0; a < 3; ++a) cnt_of[slot_of[local_of[m.facets[3 * (size_t)f + a]]]]++;
                idx.resize(tnodes.size());
                std::iota(idx.begin(), idx.end(), 0);
                std::sort(idx.begin(), idx.end(), [&](int32_t x, int32_t y) {
                    return cnt_of[x] != cnt_of[y] ? cnt_of[x] > cnt_of[y] : tnodes[x] < tnodes[y];
                });
                for (int32_t l : tnodes) slot_of[l] = -1;
                sorted.resize(tnodes.size());
                for (size_t k = 0; k < idx.size(); ++k) sorted[k] = tnodes[idx[k]];
                tnodes.swap(sorted);
                int ncsr = 0;  // each slot's list padded to a multiple of 4 (16-byte reads in the reduction)
                for (int32_t cn : cnt_of) ncsr += (cn + 3) & ~3;
                meta[t] = TileMeta{(int32_t)te.size(), (int32_t)tnodes.size(), (int32_t)tfacets.size(), ncsr};
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
    // slot order inside a tile: tile-private nodes first (by contribution count, descending: similar
    // reduction-list lengths share a warp), then the tile-shared nodes in ascending node id, so the
    // partials they write and the slot copies the update kernel writes back are laid out in the
    // update's (node) order -- whole sectors instead of scattered 16 / 8-byte accesses
    if (!(std::getenv("CF_SLOT_ORDER") && std::string(std::getenv("CF_SLOT_ORDER")) == "count")) {
#pragma omp parallel for schedule(dynamic, 256)
        for (int32_t t = 0; t < rp.n_tiles; ++t) {
            auto& tn = tile_nodes[t];
            auto mid = std::stable_partition(tn.begin(), tn.end(), [&](int32_t l) {
                return ntiles_of[l] == 1 && !shared_node[l];
            });
            std::sort(mid, tn.end());
        }
    }
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
    int64_t n_if = 0, n_bc = 0, bank_before = 0, bank_after = 0, bank_a = 0, bank_b = 0, bank_ia = 0, bank_ib = 0, bank_id_a = 0;
    const char* bank_env = std::getenv("CF_BANK_ITERS");
    // swap attempts per element after the greedy colouring (measured: 8 -> -1 % tile time for
    // +13 s setup at cfg2; off by default)
    const int bank_iters = bank_env ? std::atoi(bank_env) : 0;
    const bool bank_trace = std::getenv("CF_TRACE_SETUP") && std::atoi(std::getenv("CF_TRACE_SETUP"));
    const bool slot_order_default = !(std::getenv("CF_SLOT_ORDER") && std::string(std::getenv("CF_SLOT_ORDER")) != "node")
                                    && !(std::getenv("CF_SLOT_BANKS") && std::atoi(std::getenv("CF_SLOT_BANKS")) == 0);
#pragma omp parallel num_threads(nthr) reduction(+ : n_if, n_bc)
    {
        std::vector<int32_t> slot_of(rp.n_local, -1), tfacets;
        std::vector<int32_t> ent_off, cur, poff, eslot, sperm, tn, gmem, goff, ord, bank_of;
        std::vector<uint32_t> ent, items;
        std::vector<int32_t> gcnt;
        BankPlanner bank;
#pragma omp for schedule(dynamic, 64) reduction(+ : bank_before, bank_after, bank_a, bank_b, bank_ia, bank_ib, bank_id_a)
        for (int32_t t = 0; t < rp.n_tiles; ++t) {
            const auto& te = tiles[t];
            const TileMeta tm = rp.tile_meta[t];
            const int ne = tm.ne, ns = tm.ns, nf = tm.nf;
            const TileLayout L(tm, S.temp_dep, coords);
            uint8_t* const stg = rp.blob.data() + rp.rest_off[t];  // connectivity first, then sections >= stage
            std::memset(stg, 0, (size_t)L.staged_bytes());
            auto at = [&](int32_t off) { return stg + L.stage_of(off); };
            tn.assign(tile_nodes[t].begin(), tile_nodes[t].end());
            const auto& tnodes = tn;
            for (int k = 0; k < ns; ++k) slot_of[tn[k]] = k;
            // bank-aware numbering of the tile-private slots (their order is free: the reduction's
            // thread order is sperm, the update never sees them): phase 2a reads sTH[slot] for
            // corner q of 8 consecutive elements (the bank planner keeps such blocks together), so
            // spread each block's corner slots over the 8 bank groups (slot & 7); shared slots fixed
            if (!coords && ne >= 16 && slot_order_default) {
                int np = 0;
                while (np < ns && ntiles_of[tn[np]] == 1 && !shared_node[tn[np]]) ++np;
                if (np >= 16) {
                    const int ng = 4 * ((ne + 7) / 8);
                    goff.assign(ng + 1, 0);
                    gmem.clear();
                    for (int b0 = 0, g = 0; b0 < ne; b0 += 8)
                        for (int q = 0; q < 4; ++q, ++g) {
                            for (int i = b0; i < std::min(ne, b0 + 8); ++i) {
                                const int32_t sl = slot_of[local_of[m.tets[4 * (size_t)te[i] + q]]];
                                bool dup = false;
                                for (int k = goff[g]; k < (int)gmem.size(); ++k) dup = dup || gmem[k] == sl;
                                if (!dup) gmem.push_back(sl);
                            }
                            goff[g + 1] = (int)gmem.size();
                        }
                    // private slot (old index) -> its groups
                    std::vector<std::vector<int32_t>> pg(np);
                    for (int g = 0; g < ng; ++g)
                        for (int k = goff[g]; k < goff[g + 1]; ++k)
                            if (gmem[k] < np) pg[gmem[k]].push_back(g);
                    gcnt.assign(8 * (size_t)ng, 0);
                    for (int g = 0; g < ng; ++g)
                        for (int k = goff[g]; k < goff[g + 1]; ++k)
                            if (gmem[k] >= np) gcnt[8 * (size_t)g + (gmem[k] & 7)]++;
                    int freeb[8];
                    for (int b = 0; b < 8; ++b) freeb[b] = (np - b + 7) / 8;
                    ord.resize(np);
                    std::iota(ord.begin(), ord.end(), 0);
                    std::stable_sort(ord.begin(), ord.end(),
                                     [&](int32_t x, int32_t y) { return pg[x].size() > pg[y].size(); });
                    bank_of.assign(np, -1);
                    for (int32_t o : ord) {
                        int best = -1, bc = 1 << 30;
                        for (int b = 0; b < 8; ++b) {
                            if (!freeb[b]) continue;
                            int c = 0;
                            for (int32_t g : pg[o]) c += gcnt[8 * (size_t)g + b];
                            if (c < bc || (c == bc && freeb[b] > freeb[best])) {
                                bc = c;
                                best = b;
                            }
                        }
                        bank_of[o] = best;
                        freeb[best]--;
                        for (int32_t g : pg[o]) gcnt[8 * (size_t)g + best]++;
                    }
                    // new index: the k-th private slot of bank b gets b + 8k (stable in old order)
                    int nextb[8];
                    for (int b = 0; b < 8; ++b) nextb[b] = b;
                    std::vector<int32_t> newtn(tn.begin(), tn.begin() + np);
                    for (int o = 0; o < np; ++o) {
                        newtn[nextb[bank_of[o]]] = tn[o];
                        nextb[bank_of[o]] += 8;
                    }
                    std::copy(newtn.begin(), newtn.end(), tn.begin());
                    for (int k = 0; k < np; ++k) slot_of[tn[k]] = k;
                }
            }
            tile_facets(te, tfacets);
            // per-slot contributions in reduction order (ascending element, then facets):
            // element corner (i << 2 | q) or 0x80000000 | final 16-bit code
            ent_off.assign(ns + 1, 0);
            for (int i = 0; i < ne; ++i)
                for (int a = 0; a < 4; ++a) ent_off[slot_of[local_of[m.tets[4 * (size_t)te[i] + a]]] + 1]++;
            for (int i = 0; i < nf; ++i)
                for (int a = 0; a < 3; ++a) ent_off[slot_of[local_of[m.facets[3 * (size_t)tfacets[i] + a]]] + 1]++;
            for (int k = 0; k < ns; ++k) ent_off[k + 1] += ent_off[k];
            ent.resize(ent_off[ns]);
            {
                cur.assign(ent_off.begin(), ent_off.end() - 1);
                for (int i = 0; i < ne; ++i)
                    for (int a = 0; a < 4; ++a)
                        ent[cur[slot_of[local_of[m.tets[4 * (size_t)te[i] + a]]]]++] = (uint32_t)(i << 2 | a);
                for (int i = 0; i < nf; ++i)
                    for (int a = 0; a < 3; ++a)
                        ent[cur[slot_of[local_of[m.facets[3 * (size_t)tfacets[i] + a]]]]++] =
                            0x80000000u | L.code_facet(i, a);
            }
            // padded lists (multiples of 4: the kernel reads 4 codes at a time; padding = the zero
            // operand), then bank-aware element positions (stored layout)
            poff.assign(ns + 1, 0);
            for (int k = 0; k < ns; ++k) poff[k + 1] = poff[k] + ((ent_off[k + 1] - ent_off[k] + 3) & ~3);
            items.assign(poff[ns], 0x80000000u | L.code_zero());
            for (int k = 0; k < ns; ++k)
                std::copy(ent.begin() + ent_off[k], ent.begin() + ent_off[k + 1], items.begin() + poff[k]);
            // phase-3 thread order: slots by padded list length (descending), so a warp's reduction
            // loops have similar trip counts whatever the slot order (tile-shared slots by node id)
            sperm.resize(ns);
            std::iota(sperm.begin(), sperm.end(), 0);
            std::stable_sort(sperm.begin(), sperm.end(), [&](int32_t x, int32_t y) {
                return poff[x + 1] - poff[x] > poff[y + 1] - poff[y];
            });
            bank.sperm = sperm.data();
            eslot.resize(4 * (size_t)ne);
            for (int i = 0; i < ne; ++i)
                for (int a = 0; a < 4; ++a) eslot[4 * i + a] = slot_of[local_of[m.tets[4 * (size_t)te[i] + a]]];
            bank.run(ne, ns, eslot.data(), poff, items, coords ? 0 : bank_iters * ne, (uint64_t)t + 1);
            if (bank_trace) {
                BankPlanner id;
                id.sperm = sperm.data();
                id.run(ne, ns, eslot.data(), poff, items, 0, 0, false);  // reference-order positions
                if (!coords) {
                    bank_before += id.total_cost();
                    bank_after += bank.total_cost();
                    bank_id_a += id.total_cost(1);
                    bank_a += bank.total_cost(1);
                    bank_b += bank.total_cost(2);
                    bank_ia += bank.n_groups(1);
                    bank_ib += bank.n_groups(2);
                }
            }
            const int32_t* lp = bank.pos.data();  // element i -> local position
            uint16_t* csec = (uint16_t*)at(L.conn);  // ushort4 per element
            for (int i = 0; i < ne; ++i) {
                const int32_t e = te[i], p = lp[i];
                rp.elem_global[elem_off[t] + p] = e;
                for (int a = 0; a < 4; ++a) {
                    const int32_t l = local_of[m.tets[4 * (size_t)e + a]];  // oriented (finalize_mesh)
                    rp.tets_ord[4 * (size_t)(elem_off[t] + p) + a] = l;
                    csec[4 * p + a] = (uint16_t)slot_of[l];
                }
                *at(L.region + p) = (uint8_t)m.region[e];
            }
            for (int i = 0; i < nf; ++i) {
                const int32_t f = tfacets[i];
                const int32_t kind = S.facet_kind[f];
                uint8_t* rec = at(L.fac + 48 * i);  // (area, slots + kind), sister nodes, pad
                uint16_t* fs = (uint16_t*)(rec + 8);
                for (int a = 0; a < 3; ++a) fs[a] = (uint16_t)slot_of[local_of[m.facets[3 * (size_t)f + a]]];
                fs[3] = (uint16_t)kind;
                const double area = triangle_area(m.pos(m.facets[3 * (size_t)f]), m.pos(m.facets[3 * (size_t)f + 1]),
                                                  m.pos(m.facets[3 * (size_t)f + 2]));
                std::memcpy(rec, &area, 8);
                int32_t* sis = (int32_t*)(rec + 16);
                if (S.P.kind[kind].interface) {
                    const int32_t se = S.pairs[S.pair_of_facet[f]].sister;
                    for (int a = 0; a < 4; ++a) sis[a] = local_of[m.tets[4 * (size_t)se + a]];
                    n_if++;
                } else {
                    n_bc++;
                }
            }
            uint16_t* sp = (uint16_t*)at(L.sperm);
            for (int j = 0; j < ns; ++j) sp[j] = (uint16_t)sperm[j];
            uint16_t* cend = (uint16_t*)at(L.csr_end);
            uint16_t* csr = (uint16_t*)at(L.csr);
            int32_t* sn = (int32_t*)at(L.snode);
            const int64_t so = rp.tile_slot_off[t];
            for (int k = 0; k < (int)cf_round(ns, 2); ++k) {
                if (k >= ns) {  // padding slot (never a merge target)
                    rp.slot_node[so + k] = -1;
                    continue;
                }
                const int32_t l = tnodes[k];
                rp.slot_node[so + k] = (int32_t)(((uint32_t)rp.node_region[l] << 28) | (uint32_t)l);
                const bool priv = ntiles_of[l] == 1 && !shared_node[l];
                const bool dir = !rp.node_dir.empty() && rp.node_dir[l] >= 0;
                *at(L.sinfo + k) = (uint8_t)((rp.node_region[l] & 0x3f) | (dir ? 0x40 : 0) | (priv ? 0x80 : 0));
                for (int32_t q = poff[k]; q < poff[k + 1]; ++q) {
                    const uint32_t it = items[q];
                    csr[q] = (it & 0x80000000u) ? (uint16_t)(it & 0xffffu) : L.code_elem(lp[it >> 2], (int)(it & 3));
                }
                cend[k] = (uint16_t)poff[k + 1];
                sn[k] = l;
            }
            for (int k = 0; k < ns; ++k) slot_of[tnodes[k]] = -1;
        }
    }
    if (bank_trace)
        std::fprintf(stderr, "[cf setup] rank %d bank-aware positions: shared-memory wavefronts %lld -> %lld "
                     "(reduction reads %lld from %lld, ideal %lld; corner gathers %lld, ideal %lld)\n", rank,
                     (long long)bank_before, (long long)bank_after, (long long)bank_a, (long long)bank_id_a, (long long)bank_ia,
                     (long long)bank_b, (long long)bank_ib);
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
