// ref_bench.cpp — TEST INFRASTRUCTURE: the reference arm of bench.py (`--impl reference`) and
// the GPU arm's `cpu_baseline`, as one self-contained executable (oracle/_ref/ref_bench, built
// by oracle/Makefile from the UNMODIFIED reference headers). The process that times the
// reference loads neither the product library nor Python: the synthetic workload comes from
// the oracle's own generator (oracle/fixture.c, pinned bit for bit to the product's), the
// physics setup is BASELINE's (restated below; tests/test_oracle_pin.py checks it against
// paper_1005_3158_b200/configs.py), and the timed region is the reference's own loop:
//   pair_sister_facets (mesh.hpp:456) -> SubDomain::whole (blocked.hpp:41) ->
//   build_worker_model (:156, `blocks` cache blocks; or autotune_block_count :587-623) ->
//   init_worker_fields (:419) -> refresh_ambient (:441) -> blocked_step (:542) x steps,
// timed with steady_clock around the step loop only (solve_serial's loop_seconds, :673-684;
// setup excluded). Serial by contract: one host core.
//
// usage: ref_bench --workload cfg1..cfg5 [--window i0:i1,j0:j1,k0:k1] [--steps K] [--warmup W]
//                  [--blocks B | --autotune c1,c2,...] [--tune-steps S] [--describe] [--dump-T file]
#include <castfem/blocked.hpp>
#include <castfem/reorder.hpp>

#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../include/castfem_b200.h"

extern "C" {
int or_generate_fixture(int32_t kind, int32_t n, double radius, double jitter, uint64_t seed, uint64_t perm_seed,
                        const int32_t* window, cf_fixture* out);
double or_counter_uniform(uint64_t seed, uint64_t key);
}

using namespace castfem;

namespace {

// BASELINE.json configs as generator rules; dt_safety = 0.9 * 2/lambda_max mapped
// onto the reference's Eq. 13 bound (profiles/dt_safety_r0*.json); h_i = 1000 W/m^2K (builder's
// choice, SURVEY §0 trap 3); T0 = region pouring temperature + U(-1, 1) K per grid point.
struct Workload {
    const char* name;
    int kind, n;
    double jitter;
    uint64_t seed, perm_seed;
    double dt_safety;
    int steps;
};
const Workload kWorkloads[] = {
    {"cfg1", 0, 32, 0.0, 0, 0, 0.14417607623697684, 100},
    {"cfg2", 1, 128, 0.0, 0, 0, 0.14355290898864603, 1000},
    {"cfg3", 1, 70, 0.2, 7, 11, 0.12107620380138684, 500},
    {"cfg4", 1, 256, 0.0, 0, 0, 0.14434666132619436, 500},
    {"cfg5", 1, 512, 0.0, 0, 0, 0.14472535840047063, 200},
};
constexpr double kRadius = 0.35, kHInterface = 1000.0, kNoise = 1.0;
constexpr uint64_t kNoiseSeed = 1;

MaterialTable material(double rho, double c, double k, double L, double Ts, double Tl, double T0) {
    MaterialTable m;
    m.rho = rho;
    m.c_of_T = PiecewiseLinear::constant(c);
    m.k_of_T = PiecewiseLinear::constant(k);
    m.latent_heat = L;
    m.solidus = Ts;
    m.liquidus = Tl;
    m.initial_temperature = T0;
    m.finalize();
    return m;
}

[[noreturn]] void die(const std::string& msg) {
    std::fprintf(stderr, "ref_bench: %s\n", msg.c_str());
    std::exit(2);
}

}  // namespace

int main(int argc, char** argv) {
    std::string wl = "cfg2", dump;
    int32_t window[6];
    bool have_window = false, describe = false;
    long steps = 10, warmup = 1, blocks = 1, tune_steps = 3;
    bool rcm = false;  // RCM-reordered mesh: permute_mesh(m, rcm_permutation(build_node_graph(m)))
    std::vector<idx> candidates;
    for (int a = 1; a < argc; ++a) {
        const std::string k = argv[a];
        auto val = [&]() -> std::string {
            if (a + 1 >= argc) die("missing value for " + k);
            return argv[++a];
        };
        if (k == "--workload") wl = val();
        else if (k == "--steps") steps = std::atol(val().c_str());
        else if (k == "--warmup") warmup = std::atol(val().c_str());
        else if (k == "--blocks") blocks = std::atol(val().c_str());
        else if (k == "--tune-steps") tune_steps = std::atol(val().c_str());
        else if (k == "--describe") describe = true;
        else if (k == "--rcm") rcm = true;
        else if (k == "--dump-T") dump = val();
        else if (k == "--autotune") {
            std::string v = val();
            for (size_t p = 0; p < v.size();) {
                size_t q = v.find(',', p);
                if (q == std::string::npos) q = v.size();
                candidates.push_back((idx)std::atol(v.substr(p, q - p).c_str()));
                p = q + 1;
            }
        } else if (k == "--window") {
            const std::string v = val();
            if (std::sscanf(v.c_str(), "%d:%d,%d:%d,%d:%d", &window[0], &window[1], &window[2], &window[3], &window[4],
                            &window[5]) != 6)
                die("--window wants i0:i1,j0:j1,k0:k1");
            have_window = true;
        } else {
            die("unknown argument " + k);
        }
    }
    const Workload* W = nullptr;
    for (const Workload& w : kWorkloads)
        if (wl == w.name) W = &w;
    if (!W) die("unknown workload " + wl);

    // ---- the synthetic mesh (oracle generator) into the reference's own Mesh type
    const auto t_setup = std::chrono::steady_clock::now();
    cf_fixture fx{};
    const int32_t* win = have_window ? window : nullptr;
    if (or_generate_fixture(W->kind, W->n, kRadius, W->jitter, W->seed, W->perm_seed, win, &fx) != CF_OK)
        die("bad fixture / window");
    std::vector<double> coords(3 * (size_t)fx.n_nodes);
    std::vector<int32_t> tets(4 * (size_t)fx.n_elems), region(fx.n_elems), facets(3 * (size_t)fx.n_facets),
        ftag(fx.n_facets), grid(fx.n_nodes);
    fx.coords = coords.data();
    fx.tets = tets.data();
    fx.region = region.data();
    fx.facets = facets.data();
    fx.facet_tag = ftag.data();
    fx.node_grid = grid.data();
    if (or_generate_fixture(W->kind, W->n, kRadius, W->jitter, W->seed, W->perm_seed, win, &fx) != CF_OK)
        die("fixture generation failed");
    Mesh m;
    m.nodes.resize(fx.n_nodes);
    for (idx i = 0; i < fx.n_nodes; ++i) m.nodes[i] = {coords[3 * (size_t)i], coords[3 * (size_t)i + 1], coords[3 * (size_t)i + 2]};
    m.tets.resize(fx.n_elems);
    for (idx e = 0; e < fx.n_elems; ++e) {
        for (int q = 0; q < 4; ++q) m.tets[e].n[q] = tets[4 * (size_t)e + q];
        m.tets[e].region = region[e];
    }
    m.facets.resize(fx.n_facets);
    for (idx f = 0; f < fx.n_facets; ++f) {
        for (int q = 0; q < 3; ++q) m.facets[f].n[q] = facets[3 * (size_t)f + q];
        m.facets[f].tag = ftag[f];
    }
    m.tags = {"outer"};
    if (W->kind == 1) {
        m.tags.push_back("cast_if");
        m.tags.push_back("mold_if");
        m.contacts.push_back({1, 2});
    }
    std::vector<double>().swap(coords);
    std::vector<int32_t>().swap(tets);
    std::vector<int32_t>().swap(facets);
    finalize_mesh(m);
    if (rcm) {  // BASELINE configs[1] "RCM-reordered" (the reference's own pass, reorder.hpp:127-163)
        const auto perm = rcm_permutation(build_node_graph(m));
        m = permute_mesh(m, perm);
        std::vector<int32_t> g2(grid.size());
        for (size_t i = 0; i < grid.size(); ++i) g2[perm[i]] = grid[i];
        grid.swap(g2);
    }

    // ---- BASELINE physics
    SimulationSetup setup;
    BoundaryCondition outer;
    outer.kind = BoundaryCondition::Kind::flux;
    outer.t_inf = 300.0;
    if (W->kind == 0) {
        setup.materials.push_back(material(2700.0, 900.0, 200.0, 0.0, 0.0, 0.0, 973.0));
        outer.h = 100.0;
    } else {
        setup.materials.push_back(material(2700.0, 900.0, 200.0, 3.9e5, 821.0, 913.0, 973.0));  // Al casting
        setup.materials.push_back(material(1500.0, 1000.0, 1.0, 0.0, 0.0, 0.0, 300.0));         // sand mould
        outer.h = 20.0;
        InterfaceCoeff ic;
        ic.tag_a = "cast_if";
        ic.tag_b = "mold_if";
        ic.var = InterfaceCoeff::Var::time;
        ic.h = PiecewiseLinear::constant(kHInterface);
        setup.interface_coeffs.push_back(ic);
    }
    setup.boundary_conditions["outer"] = outer;
    setup.solver.dt_safety = W->dt_safety;
    // T0: region temperature + seeded noise per grid point (index-keyed; every node is free)
    std::vector<double> T0(fx.n_nodes);
    {
        std::vector<int32_t> node_reg(fx.n_nodes, 0);
        for (idx e = 0; e < fx.n_elems; ++e)
            for (int q = 0; q < 4; ++q) node_reg[m.tets[e].n[q]] = region[e];
        for (idx i = 0; i < fx.n_nodes; ++i)
            T0[i] = setup.materials[node_reg[i]].initial_temperature +
                    (-kNoise + (kNoise - -kNoise) * or_counter_uniform(kNoiseSeed, (uint64_t)grid[i]));
    }
    if (describe) {
        std::printf("{\"workload\": \"%s\", \"elements\": %d, \"nodes\": %d, \"facets\": %d, \"dt_safety\": %.17g, "
                    "\"h_interface\": %.17g, \"T0_sum\": %.17g}\n",
                    W->name, fx.n_elems, fx.n_nodes, fx.n_facets, W->dt_safety, kHInterface,
                    [&] { double s = 0; for (double v : T0) s += v; return s; }());
        return 0;
    }

    const std::vector<InterfacePair> pairs = pair_sister_facets(m);
    SubDomain domain = SubDomain::whole(m);
    TuneReport tune;
    double tune_seconds = 0;
    if (!candidates.empty()) {
        const auto t0 = std::chrono::steady_clock::now();
        tune = autotune_block_count(m, setup, pairs, domain, T0, candidates, (int)tune_steps, (double)steps);
        tune_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        blocks = tune.chosen;
    }
    const WorkerModel model = build_worker_model(m, setup, pairs, std::move(domain), (idx)blocks);
    WorkerFields f;
    init_worker_fields(model, setup, T0, f);
    Workspace ws(model.plan);
    refresh_ambient(model, f);
    const double setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_setup).count() - tune_seconds;

    for (long s = 0; s < warmup; ++s) blocked_step(model, setup, f, ws, 0);
    const auto begin = std::chrono::steady_clock::now();
    for (long s = 0; s < steps; ++s) blocked_step(model, setup, f, ws, 0);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - begin).count();

    double tsum = 0, tmin = f.state.T.empty() ? 0 : f.state.T[0], tmax = tmin;
    for (double v : f.state.T) {
        tsum += v;
        tmin = std::min(tmin, v);
        tmax = std::max(tmax, v);
    }
    if (!dump.empty()) {
        std::vector<double> T(m.node_count());
        for (idx i = 0; i < (idx)model.domain.nodes.size(); ++i) T[model.domain.nodes[i]] = f.state.T[i];
        FILE* fp = std::fopen(dump.c_str(), "wb");
        if (!fp || std::fwrite(T.data(), sizeof(double), T.size(), fp) != T.size()) die("cannot write " + dump);
        std::fclose(fp);
    }
    std::string cand_json = "[", sec_json = "[";
    for (size_t i = 0; i < tune.candidates.size(); ++i) {
        cand_json += (i ? ", " : "") + std::to_string(tune.candidates[i]);
        char b[64];
        std::snprintf(b, sizeof b, "%s%.6g", i ? ", " : "", tune.seconds[i]);
        sec_json += b;
    }
    cand_json += "]";
    sec_json += "]";
    std::printf("{\"workload\": \"%s\", \"rcm\": %s, \"window\": %s, \"elements\": %d, \"nodes\": %d, \"facets\": %d, "
                "\"interface_pairs\": %zu, \"blocks\": %ld, \"warmup\": %ld, \"steps\": %ld, \"seconds\": %.9g, "
                "\"setup_seconds\": %.3f, \"element_updates_per_s\": %.9g, \"dt\": %.17g, \"time\": %.17g, "
                "\"T_sum\": %.17g, \"T_min\": %.17g, \"T_max\": %.17g, \"clamp_steps\": %ld, "
                "\"autotune\": {\"candidates\": %s, \"seconds\": %s, \"tune_seconds\": %.3f}}\n",
                W->name, rcm ? "true" : "false",
                have_window ? ("\"" + std::to_string(window[0]) + ":" + std::to_string(window[1]) + "," +
                               std::to_string(window[2]) + ":" + std::to_string(window[3]) + "," +
                               std::to_string(window[4]) + ":" + std::to_string(window[5]) + "\"").c_str()
                            : "null",
                fx.n_elems, fx.n_nodes, fx.n_facets, pairs.size(), blocks, warmup, steps, secs, setup_s,
                secs > 0 ? (double)fx.n_elems * (double)steps / secs : 0.0, f.state.dt, f.state.time, tsum, tmin, tmax,
                (long)f.clamp_steps, cand_json.c_str(), sec_json.c_str(), tune_seconds);
    return 0;
}
