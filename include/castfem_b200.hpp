// castfem_b200.hpp — header-only C++ host shim over the C-ABI (castfem_b200.h)
// for users of the reference castfem API (/root/reference/proj/include/castfem/).
//
// It keeps the reference's call shapes:
//   castfem::solve_serial(mesh, setup, opts)          (blocked.hpp:650)
//     -> castfem_b200::solve_gpu(mesh, setup, opts)   same SolveResult fields
//   build_worker_model + init_worker_fields + blocked_step (blocked.hpp:156, 419, 542)
//     -> castfem_b200::Plan(mesh, setup, opts).step(n) / .fields()
// Mesh and setup are read through the reference types' public members
// (Mesh::nodes/tets/facets/tags/contacts, MaterialTable, BoundaryCondition,
// InterfaceCoeff, SolverConfig), as templates, so this header does not need
// the reference headers to compile; a castfem user passes castfem objects.
// Errors become the reference exception types when those are visible
// (CASTFEM_B200_REFERENCE_EXCEPTIONS), else castfem_b200::error.
#pragma once

#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "castfem_b200.h"

namespace castfem_b200 {

struct error : std::runtime_error {
    int code;
    error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int status) {
    if (status == CF_OK) return;
    char buf[1024];
    cf_last_error(buf, sizeof buf);
#ifdef CASTFEM_B200_REFERENCE_EXCEPTIONS
    switch (status) {
        case CF_PARSE: throw castfem::parse_error(buf, 0);
        case CF_VALIDATION: throw castfem::validation_error(buf);
        case CF_CONFIG: throw castfem::config_error(buf);
        case CF_PROTOCOL: throw castfem::protocol_error(buf);
        case CF_DEGENERATE: throw castfem::degenerate_element_error(buf);
        default: break;
    }
#endif
    throw error(status, buf);
}

struct SolveOptions {             // castfem::SolveOptions (blocked.hpp:630-636) + B200 knobs
    long max_steps = 0;
    int mode = CF_MODE_DETERMINISTIC;
    int node_order = CF_NODE_ORDER_TILE;
    int elem_order = CF_ELEM_ORDER_MORTON;
    int tile_elems = 384;
    int geometry = CF_GEOM_STORED;
    int device = 0;
    // domain decomposition (SPEC S:413-485 parallel_solve; partition.hpp:377-422): RCB parts unless
    // part_of_element (load_partmap's vector) is given. local_ranks == world_size runs every rank
    // in this process on `device` (the SPEC's mandatory in-process transport); one rank per
    // process needs a cf_comm (cf_comm_create / _peer / _host) and returns this rank's nodes.
    int world_size = 1, rank = 0, local_ranks = 1;
    const std::vector<int>* part_of_element = nullptr;
    cf_comm* comm = nullptr;
};

struct SeriesSample {
    double time, t_min, t_max;
};

struct SolveResult {              // castfem::SolveResult (blocked.hpp:638-647)
    std::vector<double> T, H;
    double end_time = 0;
    long steps = 0;
    double loop_seconds = 0;      // device time of the step loop
    std::vector<SeriesSample> series;
    long clamp_steps = 0;
    int blocks_used = 0;          // tiles
};

// Flattened copies of the caller's mesh / setup in the C-ABI layout.
class Descriptors {
  public:
    template <class MeshT, class SetupT>
    Descriptors(const MeshT& m, const SetupT& s, const std::vector<double>* T0 = nullptr) {
        coords_.reserve(3 * m.nodes.size());
        for (const auto& p : m.nodes) {
            coords_.push_back(p.x);
            coords_.push_back(p.y);
            coords_.push_back(p.z);
        }
        for (const auto& t : m.tets) {
            for (int a = 0; a < 4; ++a) tets_.push_back(t.n[a]);
            region_.push_back(t.region);
        }
        for (const auto& f : m.facets) {
            for (int a = 0; a < 3; ++a) facets_.push_back(f.n[a]);
            ftag_.push_back(f.tag);
        }
        for (const auto& t : m.tags) tag_ptrs_.push_back(t.c_str());
        for (const auto& c : m.contacts) {
            contacts_.push_back(c.tag_a);
            contacts_.push_back(c.tag_b);
        }
        md_ = cf_mesh_desc{(int32_t)m.nodes.size(), coords_.data(), (int32_t)m.tets.size(), tets_.data(),
                           region_.data(),          (int32_t)m.facets.size(), facets_.data(), ftag_.data(),
                           (int32_t)tag_ptrs_.size(), tag_ptrs_.data(), (int32_t)m.contacts.size(),
                           contacts_.data()};
        tables_.reserve(4 * s.materials.size() + 2 * s.boundary_conditions.size() + 2 * s.interface_coeffs.size() + 8);
        for (const auto& mat : s.materials)
            mats_.push_back(cf_material{mat.rho, table(mat.c_of_T), table(mat.k_of_T), mat.latent_heat, mat.solidus,
                                        mat.liquidus, mat.initial_temperature});
        for (const auto& [tag, bc] : s.boundary_conditions) {
            names_.push_back(tag);
        }
        size_t i = 0;
        for (const auto& [tag, bc] : s.boundary_conditions) {
            const bool fixed = static_cast<int>(bc.kind) == 0;  // Kind::fixed is the first enumerator
            bcs_.push_back(cf_boundary_condition{names_[i++].c_str(), fixed ? CF_BC_FIXED : CF_BC_FLUX,
                                                 table(bc.fixed_T), bc.q, bc.h, bc.t_inf});
        }
        for (const auto& ic : s.interface_coeffs)
            coeffs_.push_back(cf_interface_coeff{ic.tag_a.c_str(), ic.tag_b.c_str(),
                                                 static_cast<int>(ic.var) == 1 ? CF_VAR_TEMPERATURE : CF_VAR_TIME,
                                                 table(ic.h)});
        if (T0) {
            T0_ = *T0;
        } else if constexpr (requires { s.initial_override; }) {
            // initial_override(pos, region) (material.hpp:167-168) evaluated on the host, index-keyed
            if (s.initial_override) {
                std::vector<int32_t> node_region(m.nodes.size(), 0);
                for (const auto& t : m.tets)
                    for (int a = 0; a < 4; ++a) node_region[t.n[a]] = t.region;
                T0_.resize(m.nodes.size());
                for (size_t n = 0; n < m.nodes.size(); ++n) T0_[n] = s.initial_override(m.nodes[n], node_region[n]);
            }
        }
        for (const auto& [tag, bc] : s.boundary_conditions) {
            if constexpr (requires { bc.fixed_fn; })
                if (bc.fixed_fn) throw error(CF_CONFIG, "fixed_fn (spatial Dirichlet override) is not expressible "
                                                        "through the C-ABI; use fixed_T(t)");
        }
        sd_ = cf_setup_desc{(int32_t)mats_.size(), mats_.data(), (int32_t)bcs_.size(), bcs_.data(),
                            (int32_t)coeffs_.size(), coeffs_.data(), s.solver.dt_safety, s.solver.t_end,
                            (int64_t)s.solver.output_every, T0_.empty() ? nullptr : T0_.data()};
    }
    const cf_mesh_desc* mesh() const { return &md_; }
    const cf_setup_desc* setup() const { return &sd_; }

  private:
    template <class Table>
    cf_table table(const Table& t) {
        tables_.emplace_back(t.xs);
        const double* x = tables_.back().data();
        tables_.emplace_back(t.ys);
        return cf_table{(int32_t)t.xs.size(), x, tables_.back().data()};
    }
    std::vector<double> coords_, T0_;
    std::vector<int32_t> tets_, region_, facets_, ftag_, contacts_;
    std::vector<const char*> tag_ptrs_;
    std::vector<std::vector<double>> tables_;
    std::vector<cf_material> mats_;
    std::vector<std::string> names_;
    std::vector<cf_boundary_condition> bcs_;
    std::vector<cf_interface_coeff> coeffs_;
    cf_mesh_desc md_{};
    cf_setup_desc sd_{};
};

// A device-resident plan: build_worker_model + init_worker_fields, then
// blocked_step-granular stepping.
class Plan {
  public:
    template <class MeshT, class SetupT>
    Plan(const MeshT& m, const SetupT& s, const SolveOptions& o = {}, const std::vector<double>* T0 = nullptr)
        : n_(m.nodes.size()) {
        Descriptors d(m, s, T0);
        cf_run_opts ro{};
        ro.device = o.device;
        ro.mode = o.mode;
        ro.node_order = o.node_order;
        ro.elem_order = o.elem_order;
        ro.tile_elems = o.tile_elems;
        ro.geometry = o.geometry;
        ro.world_size = o.world_size;
        ro.rank = o.rank;
        ro.local_ranks = o.local_ranks;
        static_assert(sizeof(int) == sizeof(int32_t), "part_of_element is passed as int32");
        if (o.part_of_element) {
            if (o.part_of_element->size() != m.tets.size())
                throw error(CF_INVALID_ARG, "part_of_element needs one entry per element");
            ro.partition = CF_PARTITION_GIVEN;
            ro.part_of_element = reinterpret_cast<const int32_t*>(o.part_of_element->data());
        }
        ro.comm = o.comm;
        check(cf_plan_create(d.mesh(), d.setup(), &ro, &plan_));
    }
    ~Plan() {
        if (plan_) cf_plan_destroy(plan_);
    }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    void set_temperature(const std::vector<double>& T) { check(cf_set_temperature(plan_, T.data())); }
    void step(long n = 1, double t_end = 0) { check(cf_step(plan_, n, t_end)); }
    std::vector<SeriesSample> solve(long max_steps) {
        std::vector<double> buf(3 * 65536);
        int64_t ns = 0;
        check(cf_solve(plan_, max_steps, buf.data(), 65536, &ns));
        std::vector<SeriesSample> out;
        for (int64_t i = 0; i < ns && i < 65536; ++i) out.push_back({buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]});
        return out;
    }
    void fields(std::vector<double>& T, std::vector<double>& H) {
        T.assign(n_, 0.0);
        H.assign(n_, 0.0);
        check(cf_get_fields(plan_, T.data(), H.data()));
    }
    cf_stats stats() {
        cf_stats s{};
        check(cf_get_stats(plan_, &s));
        return s;
    }

  private:
    size_t n_;
    cf_plan* plan_ = nullptr;
};

// autotune_block_count on the B200 (blocked.hpp:558-623): the knob is elements per tile.
struct TuneReport {               // castfem::TuneReport
    std::vector<int> candidates;
    std::vector<double> seconds;  // best-of-2 device time of trial_steps per candidate (+inf: infeasible)
    int chosen = 0;
    double overhead_fraction = 0;
};

template <class MeshT, class SetupT>
TuneReport autotune_tiles(const MeshT& m, const SetupT& s, const SolveOptions& o = {},
                          std::vector<int> candidates = {}, int trial_steps = 10,
                          double projected_total_steps = 0) {
    Descriptors d(m, s);
    cf_run_opts ro{};
    ro.device = o.device;
    ro.mode = o.mode;
    ro.node_order = o.node_order;
    ro.elem_order = o.elem_order;
    ro.geometry = o.geometry;
    ro.world_size = 1;
    ro.local_ranks = 1;
    if (candidates.empty()) {
        int32_t buf[16], n = 0;
        check(cf_default_tile_candidates((int64_t)m.tets.size(), buf, 16, &n));
        candidates.assign(buf, buf + n);
    }
    std::vector<int32_t> c(candidates.begin(), candidates.end());
    TuneReport r;
    r.candidates = candidates;
    r.seconds.assign(c.size(), 0.0);
    cf_tune_report rep{};
    check(cf_autotune_tiles(d.mesh(), d.setup(), &ro, c.data(), (int32_t)c.size(), trial_steps,
                            projected_total_steps, r.seconds.data(), &rep));
    r.chosen = rep.chosen;
    r.overhead_fraction = rep.overhead_fraction;
    return r;
}

// solve_serial on the B200 (blocked.hpp:650-696): same loop semantics.
template <class MeshT, class SetupT>
SolveResult solve_gpu(const MeshT& m, const SetupT& s, const SolveOptions& o = {},
                      const std::vector<double>* T0 = nullptr) {
    Plan p(m, s, o, T0);
    SolveResult r;
    r.series = p.solve(o.max_steps);
    p.fields(r.T, r.H);
    const cf_stats st = p.stats();
    r.end_time = st.time;
    r.steps = (long)st.step_index;
    r.loop_seconds = st.loop_seconds;
    r.clamp_steps = (long)st.clamp_steps;
    r.blocks_used = st.n_tiles;
    return r;
}

}  // namespace castfem_b200
