/* Plain-C caller of the C-ABI (include/castfem_b200.h): a Kuhn cube of 6 tets with a convective
 * skin, phase change and a temperature-dependent c(T), described with hand-filled descriptors --
 * no C++, no Python. Runs 25 steps in deterministic mode twice (stored and coordinates layouts)
 * and prints the nodal temperatures as hex doubles; tests/test_gpu_edge.py::test_plain_c_caller
 * builds it, runs it on the GPU box and compares the output bit for bit with the oracle. */
#include <stdio.h>
#include <string.h>

#include "castfem_b200.h"

static int fail(const char* what, int status) {
    char msg[512];
    cf_last_error(msg, sizeof msg);
    fprintf(stderr, "%s: status %d: %s\n", what, status, msg);
    return 1;
}

int main(void) {
    /* unit cube, nodes numbered x fastest; the six Kuhn tets around the main diagonal 0-7 */
    const double coords[8 * 3] = {0, 0, 0, 1, 0, 0, 0, 1, 0, 1, 1, 0, 0, 0, 1, 1, 0, 1, 0, 1, 1, 1, 1, 1};
    const int32_t tets[6 * 4] = {0, 1, 3, 7, 0, 1, 5, 7, 0, 2, 3, 7, 0, 2, 6, 7, 0, 4, 5, 7, 0, 4, 6, 7};
    const int32_t region[6] = {0, 0, 0, 0, 0, 0};
    /* the 12 boundary triangles (two per cube face) */
    const int32_t facets[12 * 3] = {0, 1, 3, 0, 2, 3, 4, 5, 7, 4, 6, 7, 0, 1, 5, 0, 4, 5,
                                    2, 3, 7, 2, 6, 7, 0, 2, 6, 0, 4, 6, 1, 3, 7, 1, 5, 7};
    const int32_t facet_tag[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const char* tags[1] = {"skin"};
    cf_mesh_desc mesh;
    memset(&mesh, 0, sizeof mesh);
    mesh.n_nodes = 8;
    mesh.coords = coords;
    mesh.n_elems = 6;
    mesh.tets = tets;
    mesh.region = region;
    mesh.n_facets = 12;
    mesh.facets = facets;
    mesh.facet_tag = facet_tag;
    mesh.n_tags = 1;
    mesh.tags = tags;

    const double cx[2] = {300.0, 1000.0}, cy[2] = {850.0, 1100.0}, kx[1] = {0.0}, ky[1] = {200.0};
    cf_material mat;
    memset(&mat, 0, sizeof mat);
    mat.rho = 2700.0;
    mat.c.n = 2, mat.c.x = cx, mat.c.y = cy;
    mat.k.n = 1, mat.k.x = kx, mat.k.y = ky;
    mat.latent_heat = 3.9e5;
    mat.solidus = 821.0;
    mat.liquidus = 913.0;
    mat.initial_temperature = 930.0;
    cf_boundary_condition bc;
    memset(&bc, 0, sizeof bc);
    bc.tag = "skin";
    bc.kind = CF_BC_FLUX;
    bc.h = 50.0;
    bc.t_inf = 300.0;
    const double T0[8] = {930.0, 925.0, 921.5, 917.0, 912.0, 908.5, 903.0, 899.0};
    cf_setup_desc setup;
    memset(&setup, 0, sizeof setup);
    setup.n_materials = 1;
    setup.materials = &mat;
    setup.n_bcs = 1;
    setup.bcs = &bc;
    setup.dt_safety = 0.002;
    setup.initial_T = T0;

    for (int geometry = 0; geometry < 2; ++geometry) {
        cf_run_opts opts;
        memset(&opts, 0, sizeof opts);
        opts.mode = CF_MODE_DETERMINISTIC;
        opts.node_order = CF_NODE_ORDER_TILE;
        opts.elem_order = CF_ELEM_ORDER_MORTON;
        opts.tile_elems = 4; /* two tiles: shared nodes go through the merge */
        opts.world_size = 1;
        opts.local_ranks = 1;
        opts.geometry = geometry ? CF_GEOM_COORDS : CF_GEOM_STORED;
        cf_plan* plan = NULL;
        int st = cf_plan_create(&mesh, &setup, &opts, &plan);
        if (st != CF_OK) return fail("cf_plan_create", st);
        if ((st = cf_step(plan, 25, 0.0)) != CF_OK) return fail("cf_step", st);
        double T[8], H[8];
        if ((st = cf_get_fields(plan, T, H)) != CF_OK) return fail("cf_get_fields", st);
        cf_stats stats;
        if ((st = cf_get_stats(plan, &stats)) != CF_OK) return fail("cf_get_stats", st);
        printf("geometry %d steps %lld tiles %d time %a\n", geometry, (long long)stats.step_index, stats.n_tiles, stats.time);
        for (int i = 0; i < 8; ++i) printf("T %d %a %a\n", i, T[i], H[i]);
        cf_plan_destroy(plan);
    }
    /* the error path: a facet tag left without a condition is a configuration error, reported with the
     * reference's message (resolve_facet_tag blocked.hpp:127-149) */
    bc.tag = "nope";
    cf_run_opts opts;
    memset(&opts, 0, sizeof opts);
    opts.world_size = opts.local_ranks = 1;
    cf_plan* plan = NULL;
    const int st = cf_plan_create(&mesh, &setup, &opts, &plan);
    char msg[256];
    cf_last_error(msg, sizeof msg);
    printf("bad tag: status %d: %s\n", st, msg);
    return st == CF_OK;
}
