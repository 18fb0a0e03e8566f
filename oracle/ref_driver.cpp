// ref_driver.cpp — TEST INFRASTRUCTURE: a thin extern "C" driver around the
// UNMODIFIED reference headers (/root/reference/proj/include/castfem/), built
// by oracle/Makefile into oracle/_ref/libcastfem_ref.so (git-ignored; it
// travels to the GPU box as a binary). No reference source is copied: this
// file only converts the boundary structs of include/castfem_b200.h into the
// reference's own types and calls its public API:
//   finalize_mesh (mesh.hpp:148), pair_sister_facets (mesh.hpp:456),
//   initial_temperatures (blocked.hpp:396), build_worker_model (:156),
//   init_worker_fields (:419), refresh_ambient (:441), blocked_step (:542),
//   rcm_permutation / bandwidth / build_node_graph (reorder.hpp:17-148),
//   tet_geometry (geometry.hpp:48), MaterialTable::enthalpy (material.hpp:89),
//   apparent_heat_capacity (fem.hpp:26).
// The stepping loop mirrors solve_serial (blocked.hpp:650-696) but takes an
// index-keyed T0, which solve_serial's position-keyed
// initial_override hook cannot express for duplicated interface nodes.
#include <castfem/blocked.hpp>
#include <castfem/partition.hpp>
#include <castfem/reorder.hpp>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>

#include "../include/castfem_b200.h"

using namespace castfem;

namespace {

thread_local std::string g_err;

int map_exception() {
    try {
        throw;
    } catch (const parse_error& e) {
        g_err = e.what();
        return CF_PARSE;
    } catch (const degenerate_element_error& e) {
        g_err = e.what();
        return CF_DEGENERATE;
    } catch (const validation_error& e) {
        g_err = e.what();
        return CF_VALIDATION;
    } catch (const config_error& e) {
        g_err = e.what();
        return CF_CONFIG;
    } catch (const protocol_error& e) {
        g_err = e.what();
        return CF_PROTOCOL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CF_INVALID_ARG;
    }
}

PiecewiseLinear to_table(const cf_table& t) {
    PiecewiseLinear p;
    for (int i = 0; i < t.n; ++i) {
        p.xs.push_back(t.x[i]);
        p.ys.push_back(t.y[i]);
    }
    return p;
}

Mesh to_mesh(const cf_mesh_desc* d, bool finalize = true) {
    Mesh m;
    m.nodes.resize(d->n_nodes);
    for (idx i = 0; i < d->n_nodes; ++i)
        m.nodes[i] = {d->coords[3 * (size_t)i], d->coords[3 * (size_t)i + 1], d->coords[3 * (size_t)i + 2]};
    m.tets.resize(d->n_elems);
    for (idx e = 0; e < d->n_elems; ++e) {
        for (int a = 0; a < 4; ++a) m.tets[e].n[a] = d->tets[4 * (size_t)e + a];
        m.tets[e].region = d->region[e];
    }
    for (idx t = 0; t < d->n_tags; ++t) m.tags.emplace_back(d->tags[t]);
    m.facets.resize(d->n_facets);
    for (idx f = 0; f < d->n_facets; ++f) {
        for (int a = 0; a < 3; ++a) m.facets[f].n[a] = d->facets[3 * (size_t)f + a];
        m.facets[f].tag = d->facet_tag[f];
    }
    for (idx c = 0; c < d->n_contacts; ++c) m.contacts.push_back({d->contacts[2 * c], d->contacts[2 * c + 1]});
    if (finalize) finalize_mesh(m);
    return m;
}

MaterialTable to_material(const cf_material& c) {
    MaterialTable m;
    m.rho = c.rho;
    m.c_of_T = to_table(c.c);
    m.k_of_T = to_table(c.k);
    m.latent_heat = c.latent_heat;
    m.solidus = c.solidus;
    m.liquidus = c.liquidus;
    m.initial_temperature = c.initial_temperature;
    return m;
}

SimulationSetup to_setup(const cf_setup_desc* s) {
    SimulationSetup setup;
    for (int i = 0; i < s->n_materials; ++i) {
        setup.materials.push_back(to_material(s->materials[i]));
        if (setup.materials.back().rho > 0) setup.materials.back().finalize();
    }
    for (int i = 0; i < s->n_bcs; ++i) {
        const auto& b = s->bcs[i];
        BoundaryCondition bc;
        bc.kind = b.kind == CF_BC_FIXED ? BoundaryCondition::Kind::fixed : BoundaryCondition::Kind::flux;
        if (b.fixed_T.n > 0) bc.fixed_T = to_table(b.fixed_T);
        bc.q = b.q;
        bc.h = b.h;
        bc.t_inf = b.t_inf;
        setup.boundary_conditions[b.tag] = bc;
    }
    for (int i = 0; i < s->n_coeffs; ++i) {
        const auto& c = s->coeffs[i];
        InterfaceCoeff ic;
        ic.tag_a = c.tag_a;
        ic.tag_b = c.tag_b;
        ic.var = c.var == CF_VAR_TEMPERATURE ? InterfaceCoeff::Var::temperature : InterfaceCoeff::Var::time;
        ic.h = to_table(c.h);
        ic.h.validate("interface h");
        setup.interface_coeffs.push_back(ic);
    }
    if (!(s->dt_safety > 0 && s->dt_safety <= 1)) throw config_error("safety must be in (0, 1]");
    setup.solver.dt_safety = s->dt_safety;
    setup.solver.t_end = s->t_end;
    setup.solver.output_every = s->output_every;
    return setup;
}

// initial_temperatures with an index-keyed override: the reference hook is
// keyed by position, so mark every node NaN through it, then fill the
// non-fixed ones from the caller's array (fixed nodes keep f(x, 0)).
std::vector<double> initial_field(const Mesh& m, SimulationSetup& setup, const double* T0) {
    if (!T0) return initial_temperatures(m, setup);
    setup.initial_override = [](const Vec3&, idx) { return std::numeric_limits<double>::quiet_NaN(); };
    std::vector<double> T = initial_temperatures(m, setup);
    setup.initial_override = nullptr;
    for (idx n = 0; n < m.node_count(); ++n)
        if (std::isnan(T[n])) T[n] = T0[n];
    return T;
}

struct RefRun {
    Mesh mesh;
    SimulationSetup setup;
    std::vector<InterfacePair> pairs;
    std::unique_ptr<WorkerModel> model;
    WorkerFields f;
    std::unique_ptr<Workspace> ws;
};

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() { return g_err.c_str(); }

// Full solve like solve_serial; stats = {time, dt, steps, clamp_steps, loop_seconds, static_dt, n_blocks}
__attribute__((visibility("default"))) int ref_solve(const cf_mesh_desc* md, const cf_setup_desc* sd,
                                                     int32_t blocks, int64_t max_steps, double* T_out,
                                                     double* H_out, double* stats, int32_t* block_map_out,
                                                     double* series, int64_t series_cap, int64_t* n_series) {
    try {
        RefRun r;
        r.mesh = to_mesh(md);
        r.setup = to_setup(sd);
        r.pairs = pair_sister_facets(r.mesh);
        SubDomain domain = SubDomain::whole(r.mesh);
        const std::vector<double> T0 = initial_field(r.mesh, r.setup, sd->initial_T);
        const WorkerModel model = build_worker_model(r.mesh, r.setup, r.pairs, std::move(domain), blocks);
        WorkerFields f;
        init_worker_fields(model, r.setup, T0, f);
        Workspace ws(model.plan);
        refresh_ambient(model, f);
        const double t_end = r.setup.solver.t_end;
        int64_t ns = 0;
        const auto begin = std::chrono::steady_clock::now();
        while ((max_steps > 0 && f.state.step_index < max_steps) ||
               (max_steps <= 0 && f.state.time < t_end)) {
            const double remaining = max_steps > 0 ? 0 : t_end - f.state.time;
            blocked_step(model, r.setup, f, ws, remaining);
            if (r.setup.solver.output_every > 0 && f.state.step_index % r.setup.solver.output_every == 0) {
                const auto [lo, hi] = std::minmax_element(f.state.T.begin(), f.state.T.end());
                if (series && ns < series_cap) {
                    series[3 * ns] = f.state.time;
                    series[3 * ns + 1] = *lo;
                    series[3 * ns + 2] = *hi;
                }
                ++ns;
            }
        }
        const double loop = std::chrono::duration<double>(std::chrono::steady_clock::now() - begin).count();
        for (idx i = 0; i < static_cast<idx>(model.domain.nodes.size()); ++i) {
            if (T_out) T_out[model.domain.nodes[i]] = f.state.T[i];
            if (H_out) H_out[model.domain.nodes[i]] = f.state.H[i];
        }
        if (stats) {
            stats[0] = f.state.time;
            stats[1] = f.state.dt;
            stats[2] = (double)f.state.step_index;
            stats[3] = (double)f.clamp_steps;
            stats[4] = loop;
            stats[5] = model.local_static_dt;
            stats[6] = (double)model.plan.blocks.size();
        }
        if (block_map_out)
            for (idx i = 0; i < (idx)model.domain.elements.size(); ++i)
                block_map_out[model.domain.elements[i]] = model.plan.block_map.part_of_element[i];
        if (n_series) *n_series = ns;
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

// Bench handle: setup once, then time blocked_step batches (loop_seconds semantics).
__attribute__((visibility("default"))) void* ref_bench_create(const cf_mesh_desc* md, const cf_setup_desc* sd) {
    try {
        auto* r = new RefRun;
        r->mesh = to_mesh(md);
        r->setup = to_setup(sd);
        r->pairs = pair_sister_facets(r->mesh);
        SubDomain domain = SubDomain::whole(r->mesh);
        const std::vector<double> T0 = initial_field(r->mesh, r->setup, sd->initial_T);
        r->model = std::make_unique<WorkerModel>(build_worker_model(r->mesh, r->setup, r->pairs, std::move(domain), 1));
        init_worker_fields(*r->model, r->setup, T0, r->f);
        r->ws = std::make_unique<Workspace>(r->model->plan);
        refresh_ambient(*r->model, r->f);
        return r;
    } catch (...) {
        map_exception();
        return nullptr;
    }
}
// Returns the loop seconds, or -status on a reference exception.
__attribute__((visibility("default"))) double ref_bench_steps(void* h, int64_t n) {
    auto* r = static_cast<RefRun*>(h);
    try {
        const auto begin = std::chrono::steady_clock::now();
        for (int64_t s = 0; s < n; ++s) blocked_step(*r->model, r->setup, r->f, *r->ws, 0);
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - begin).count();
    } catch (...) {
        return -(double)map_exception();
    }
}
__attribute__((visibility("default"))) void ref_bench_get_T(void* h, double* T_out) {
    auto* r = static_cast<RefRun*>(h);
    for (idx i = 0; i < static_cast<idx>(r->model->domain.nodes.size()); ++i)
        T_out[r->model->domain.nodes[i]] = r->f.state.T[i];
}
__attribute__((visibility("default"))) void ref_bench_destroy(void* h) { delete static_cast<RefRun*>(h); }

__attribute__((visibility("default"))) int ref_pair_sister_facets(const cf_mesh_desc* md, int32_t* out, int64_t cap,
                                                                  int64_t* n) {
    try {
        Mesh m = to_mesh(md);
        auto pairs = pair_sister_facets(m);
        *n = (int64_t)pairs.size();
        if (out)
            for (size_t i = 0; i < pairs.size() && (int64_t)i < cap; ++i) {
                out[3 * i] = pairs[i].facet;
                out[3 * i + 1] = pairs[i].sister;
                out[3 * i + 2] = pairs[i].contact;
            }
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

__attribute__((visibility("default"))) int ref_finalize(const cf_mesh_desc* md, int32_t* tets_out, int32_t* owner_out) {
    try {
        Mesh m = to_mesh(md);
        for (idx e = 0; e < m.element_count(); ++e)
            for (int a = 0; a < 4; ++a) tets_out[4 * (size_t)e + a] = m.tets[e].n[a];
        for (idx f = 0; f < (idx)m.facets.size(); ++f) owner_out[f] = m.facets[f].owner;
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

__attribute__((visibility("default"))) int ref_rcm_permutation(const cf_mesh_desc* md, int32_t seed, int32_t* out) {
    try {
        Mesh m = to_mesh(md, false);
        const AdjacencyGraph g = build_node_graph(m);
        std::optional<idx> s;
        if (seed >= 0) s = seed;
        const Permutation p = rcm_permutation(g, s);
        std::memcpy(out, p.data(), sizeof(int32_t) * p.size());
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

__attribute__((visibility("default"))) int ref_bandwidth(const cf_mesh_desc* md, const int32_t* perm, int64_t* out) {
    try {
        Mesh m = to_mesh(md, false);
        const AdjacencyGraph g = build_node_graph(m);
        Permutation p = perm ? Permutation(perm, perm + m.node_count()) : identity_permutation(m.node_count());
        *out = bandwidth(g, p);
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

__attribute__((visibility("default"))) int ref_tet_geometry(const double* p, double* out) {
    try {
        const TetGeometry g = tet_geometry({p[0], p[1], p[2]}, {p[3], p[4], p[5]}, {p[6], p[7], p[8]},
                                           {p[9], p[10], p[11]});
        out[0] = g.volume;
        for (int a = 0; a < 4; ++a) {
            out[1 + 3 * a] = g.grad[a].x;
            out[2 + 3 * a] = g.grad[a].y;
            out[3 + 3 * a] = g.grad[a].z;
        }
        out[13] = g.min_edge;
        out[14] = g.max_edge;
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

__attribute__((visibility("default"))) double ref_enthalpy(const cf_material* c, double T) {
    MaterialTable m = to_material(*c);
    m.finalize();
    return m.enthalpy(T);
}

__attribute__((visibility("default"))) double ref_apparent_heat_capacity(const double* g15, const double* Tn,
                                                                         const double* Hn, const cf_material* c) {
    MaterialTable m = to_material(*c);
    m.finalize();
    TetGeometry g;
    g.volume = g15[0];
    for (int a = 0; a < 4; ++a) g.grad[a] = {g15[1 + 3 * a], g15[2 + 3 * a], g15[3 + 3 * a]};
    g.min_edge = g15[13];
    g.max_edge = g15[14];
    return apparent_heat_capacity(g, Tn, Hn, m);
}

// ---- text formats (tests/test_io.py): the reference's own parsers
static void put_text(const std::string& s, char* out, int64_t cap, int64_t* len) {
    if (len) *len = (int64_t)s.size();
    if (out && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), (size_t)cap - 1);
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
}

// parse_mesh then write_mesh: the finalized mesh as text
__attribute__((visibility("default"))) int ref_mesh_roundtrip(const char* text, int64_t len, char* out, int64_t cap,
                                                              int64_t* out_len) {
    try {
        std::istringstream in(std::string(text, (size_t)len));
        const Mesh m = parse_mesh(in);
        std::ostringstream os;
        write_mesh(m, os);
        put_text(os.str(), out, cap, out_len);
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

static std::string g17(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}
static std::string table_text(const PiecewiseLinear& t) {
    std::string s = "[";
    for (size_t i = 0; i < t.xs.size(); ++i) s += (i ? "," : "") + g17(t.xs[i]) + ":" + g17(t.ys[i]);
    return s + "]";
}

// parse_config, dumped canonically (the Python test formats the product's parse the same way)
__attribute__((visibility("default"))) int ref_config_dump(const char* text, int64_t len, char* out, int64_t cap,
                                                           int64_t* out_len) {
    try {
        std::istringstream in(std::string(text, (size_t)len));
        const SimulationSetup S = parse_config(in);
        std::string s;
        for (size_t i = 0; i < S.materials.size(); ++i) {
            const auto& m = S.materials[i];
            s += "material " + std::to_string(i) + " rho=" + g17(m.rho) + " c=" + table_text(m.c_of_T) +
                 " k=" + table_text(m.k_of_T) + " L=" + g17(m.latent_heat) + " Ts=" + g17(m.solidus) +
                 " Tl=" + g17(m.liquidus) + " T0=" + g17(m.initial_temperature) + "\n";
        }
        for (const auto& [tag, b] : S.boundary_conditions)
            s += "bc " + tag + " kind=" + (b.kind == BoundaryCondition::Kind::fixed ? "fixed" : "flux") +
                 " T=" + table_text(b.fixed_T) + " q=" + g17(b.q) + " h=" + g17(b.h) + " t_inf=" + g17(b.t_inf) +
                 "\n";
        for (const auto& c : S.interface_coeffs)
            s += "interface " + c.tag_a + " " + c.tag_b + " var=" +
                 (c.var == InterfaceCoeff::Var::temperature ? "temperature" : "time") + " h=" + table_text(c.h) +
                 "\n";
        s += "solver safety=" + g17(S.solver.dt_safety) + " t_end=" + g17(S.solver.t_end) +
             " output_every=" + std::to_string(S.solver.output_every) + "\n";
        put_text(s, out, cap, out_len);
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

__attribute__((visibility("default"))) int ref_load_partmap(const char* text, int64_t len, int32_t n_elems,
                                                            int32_t* out, int32_t* count) {
    try {
        std::istringstream in(std::string(text, (size_t)len));
        const PartMap pm = load_partmap(in, n_elems);
        for (idx e = 0; e < n_elems; ++e) out[e] = pm.part_of_element[e];
        *count = pm.part_count;
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

// partition_elements(augment_virtual_elements(...)) (partition.hpp:43-91, 236-241) or plain
// partition_graph over build_dual_graph (augment == 0)
__attribute__((visibility("default"))) int ref_partition(const cf_mesh_desc* md, int32_t k, double tol,
                                                         int32_t augment, int32_t* out) {
    try {
        const Mesh m = to_mesh(md);
        PartMap pm;
        if (augment) {
            const auto pairs = pair_sister_facets(m);
            pm = partition_elements(augment_virtual_elements(m, pairs), k, tol);
        } else {
            const AdjacencyGraph g = build_dual_graph(m);
            pm = partition_graph(g, {}, k, tol);
        }
        for (idx e = 0; e < m.element_count(); ++e) out[e] = pm.part_of_element[e];
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}
__attribute__((visibility("default"))) int ref_partition_metrics(const cf_mesh_desc* md, const int32_t* part,
                                                                 int32_t k, int64_t* cut, double* imb,
                                                                 int32_t* nb, int64_t* split) {
    try {
        const Mesh m = to_mesh(md);
        PartMap pm;
        pm.part_count = k;
        pm.part_of_element.assign(part, part + m.element_count());
        const PartitionQuality q = partition_metrics(build_dual_graph(m), pm);
        *cut = q.edge_cut;
        *imb = q.imbalance;
        for (idx p = 0; p < k; ++p) nb[p] = q.neighbor_counts[p];
        *split = count_split_interface_pairs(m, pair_sister_facets(m), pm);
        return CF_OK;
    } catch (...) {
        return map_exception();
    }
}

}  // extern "C"
