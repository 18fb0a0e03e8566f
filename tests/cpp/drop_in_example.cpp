// Drop-in example: a castfem (reference) user calls castfem_b200::solve_gpu
// with the reference's own Mesh / SimulationSetup objects and compares it to
// castfem::solve_serial on the same input. Built by oracle/Makefile (it needs
// the reference headers) into oracle/_ref/drop_in_example; run by
// tests/test_gpu_parity.py::test_cpp_drop_in_example on a GPU box.
#include <castfem/blocked.hpp>
#define CASTFEM_B200_REFERENCE_EXCEPTIONS
#include "castfem_b200.hpp"

#include <cmath>
#include <cstdio>

using namespace castfem;

int main() {
    // 6^3-cell Kuhn cube (6 tets per cell), two regions split at x = 0.5 would share
    // nodes, so one region with a convective boundary + a time-dependent Dirichlet face
    const int n = 6;
    Mesh m;
    auto id = [&](int i, int j, int k) { return (k * (n + 1) + j) * (n + 1) + i; };
    for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) m.nodes.push_back({i / (double)n, j / (double)n, k / (double)n});
    const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const idx outer = m.add_tag("outer"), hot = m.add_tag("hot");
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                for (auto& p : perm) {
                    int v[4][3] = {{i, j, k}, {i, j, k}, {i, j, k}, {i + 1, j + 1, k + 1}};
                    v[1][p[0]] += 1;
                    v[2][p[0]] += 1;
                    v[2][p[1]] += 1;
                    Tetra t;
                    for (int q = 0; q < 4; ++q) t.n[q] = id(v[q][0], v[q][1], v[q][2]);
                    m.tets.push_back(t);
                    // boundary faces: low face of axis p[2], high face of axis p[0]
                    int lo[3] = {i, j, k}, hi[3] = {i, j, k};
                    lo[p[2]] -= 1;
                    hi[p[0]] += 1;
                    if (lo[p[2]] < 0) m.facets.push_back({{t.n[0], t.n[1], t.n[2]}, -1, p[2] == 0 ? hot : outer});
                    if (hi[p[0]] >= n) m.facets.push_back({{t.n[1], t.n[2], t.n[3]}, -1, outer});
                }
    finalize_mesh(m);
    SimulationSetup s;
    MaterialTable mat;
    mat.rho = 7800;
    mat.c_of_T = {{300.0, 900.0}, {450.0, 700.0}};
    mat.k_of_T = PiecewiseLinear::constant(45.0);
    mat.latent_heat = 2.0e5;
    mat.solidus = 700;
    mat.liquidus = 760;
    mat.initial_temperature = 650;
    mat.finalize();
    s.materials.push_back(mat);
    BoundaryCondition conv;
    conv.h = 50;
    conv.t_inf = 300;
    s.boundary_conditions["outer"] = conv;
    BoundaryCondition fixed;
    fixed.kind = BoundaryCondition::Kind::fixed;
    fixed.fixed_T = {{0.0, 200.0}, {650.0, 950.0}};
    s.boundary_conditions["hot"] = fixed;
    s.solver.dt_safety = 0.1;
    s.solver.output_every = 5;
    s.initial_override = [](const Vec3& p, idx) { return 640.0 + 20.0 * p.x * p.y; };

    SolveOptions ro;
    ro.max_steps = 40;
    const SolveResult ref = solve_serial(m, s, ro);
    castfem_b200::SolveOptions go;
    go.max_steps = 40;
    const castfem_b200::SolveResult gpu = castfem_b200::solve_gpu(m, s, go);
    double worst = 0;
    for (size_t i = 0; i < ref.T.size(); ++i) worst = std::max(worst, std::fabs(gpu.T[i] - ref.T[i]) / std::fabs(ref.T[i]));
    const bool ok = worst <= 1e-9 && gpu.steps == ref.steps && gpu.end_time == ref.end_time &&
                    gpu.series.size() == ref.series.size() && gpu.clamp_steps == ref.clamp_steps;
    std::printf("drop_in_example: nodes=%zu steps=%ld end_time=%.17g max_rel=%.3e series=%zu clamp=%ld %s\n",
                ref.T.size(), gpu.steps, gpu.end_time, worst, gpu.series.size(), gpu.clamp_steps, ok ? "OK" : "MISMATCH");
    // reference exception taxonomy through the shim
    try {
        SimulationSetup bad = s;
        bad.solver.dt_safety = 2.0;
        castfem_b200::solve_gpu(m, bad, go);
        return 2;
    } catch (const config_error&) {
    }
    // autotune_block_count recast through the shim: every candidate timed, the fastest chosen
    const castfem_b200::TuneReport tr = castfem_b200::autotune_tiles(m, s, go, {64, 128}, 3);
    const bool tune_ok = tr.candidates.size() == 2 && (tr.chosen == 64 || tr.chosen == 128) &&
                         tr.seconds[0] > 0 && tr.seconds[1] > 0;
    std::printf("autotune: chosen %d (%.3e s, %.3e s) %s\n", tr.chosen, tr.seconds[0], tr.seconds[1],
                tune_ok ? "OK" : "BAD");
    // non-overlapped element decomposition through the shim: 3 ranks in this
    // process (the in-process transport), RCB parts and a given part map, vs solve_serial
    bool dd_ok = true;
    for (int given = 0; given < 2; ++given) {
        castfem_b200::SolveOptions dd = go;
        dd.world_size = dd.local_ranks = 3;
        dd.tile_elems = 128;
        std::vector<int> parts(m.tets.size());
        for (size_t e = 0; e < parts.size(); ++e) parts[e] = (int)(e % 3);  // scattered: every node shared
        if (given) dd.part_of_element = &parts;
        const castfem_b200::SolveResult r3 = castfem_b200::solve_gpu(m, s, dd);
        double w3 = 0;
        for (size_t i = 0; i < ref.T.size(); ++i) w3 = std::max(w3, std::fabs(r3.T[i] - ref.T[i]) / std::fabs(ref.T[i]));
        const bool k = w3 <= 1e-9 && r3.steps == ref.steps && r3.end_time == ref.end_time &&
                       r3.clamp_steps == ref.clamp_steps;
        std::printf("decomposed (3 ranks, %s): max_rel=%.3e %s\n", given ? "given parts" : "RCB", w3, k ? "OK" : "MISMATCH");
        dd_ok = dd_ok && k;
    }
    return ok && tune_ok && dd_ok ? 0 : 1;
}
