/* A plain C99 consumer of include/nestrack.h (test program, built and run by
 * tests/test_c_consumer.py; no GPU needed).
 *
 * 1. Prints sizeof / offsetof of every struct the header defines, as one JSON object, so that the
 *    test can check the Python ctypes mirrors (paper_2406_13849_b200/__init__.py) against the
 *    compiler's layout.
 * 2. Links libnestrack.so and builds the C1 pincell through the builder calls with a host-only
 *    finalize (device = -1), checks the model info and a few error paths (status codes and
 *    nt_last_error), and prints them.
 */
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "nestrack.h"

#define OFF(T, f) printf("\"%s.%s\": %zu, ", #T, #f, offsetof(T, f))
#define SZ(T) printf("\"sizeof.%s\": %zu, ", #T, sizeof(T))

static int fail(const char* what, nt_status st) {
    printf("\"error\": \"%s: status %d: %s\"}\n", what, (int)st, nt_last_error());
    return 1;
}

int main(void) {
    printf("{");
    SZ(nt_build_opts); OFF(nt_build_opts, device); OFF(nt_build_opts, bih_max_leaf); OFF(nt_build_opts, pseudo_array);
    OFF(nt_build_opts, sah_ct); OFF(nt_build_opts, sah_ci);
    SZ(nt_model_info); OFF(nt_model_info, n_surfaces); OFF(nt_model_info, max_depth);
    OFF(nt_model_info, rect_specialisable); OFF(nt_model_info, rect_levels); OFF(nt_model_info, n_bih_nodes);
    OFF(nt_model_info, out_len); OFF(nt_model_info, device_bytes); OFF(nt_model_info, mesh_bins);
    OFF(nt_model_info, n_instances); OFF(nt_model_info, max_sites);
    SZ(nt_run); OFF(nt_run, seed); OFF(nt_run, pid_begin); OFF(nt_run, n); OFF(nt_run, src_lo); OFF(nt_run, src_hi);
    OFF(nt_run, max_segments); OFF(nt_run, tracker); OFF(nt_run, flags); OFF(nt_run, block_dim); OFF(nt_run, blocks_per_sm);
    SZ(nt_outputs); OFF(nt_outputs, out); OFF(nt_outputs, pflags); OFF(nt_outputs, pnseg); OFF(nt_outputs, pterm);
    OFF(nt_outputs, trace); OFF(nt_outputs, trace_cap); OFF(nt_outputs, trace_count); OFF(nt_outputs, mesh);
    OFF(nt_outputs, inst); OFF(nt_outputs, bank); OFF(nt_outputs, bank_n);
    SZ(nt_trace_rec); OFF(nt_trace_rec, pid); OFF(nt_trace_rec, s); OFF(nt_trace_rec, seg); OFF(nt_trace_rec, cell_before);
    OFF(nt_trace_rec, cell_after); OFF(nt_trace_rec, j); OFF(nt_trace_rec, kind); OFF(nt_trace_rec, level);
    OFF(nt_trace_rec, terminal); OFF(nt_trace_rec, pad); OFF(nt_trace_rec, flags);
    printf("\"abi_version\": %d, ", (int)nt_abi_version());

    /* C1 pincell (fuel / gap / clad / water) in a reflective box, host-only build */
    nt_model* m = NULL;
    nt_status st = nt_model_create(&m);
    if (st != NT_OK) return fail("create", st);
    const double hp = 0.63, h = 365.76;
    const double planes[6] = {-hp, hp, -hp, hp, 0.0, h};
    const nt_surface_kind pk[6] = {NT_PX, NT_PX, NT_PY, NT_PY, NT_PZ, NT_PZ};
    int32_t sid[9], mat[4], root, pin, cell, id;
    for (int k = 0; k < 6; ++k) {
        double c[4] = {planes[k], 0, 0, 0};
        if ((st = nt_add_surface(m, pk[k], c, NT_BC_REFLECT, &sid[k])) != NT_OK) return fail("surface", st);
    }
    const double radii[3] = {0.4096, 0.4180, 0.4750};
    for (int k = 0; k < 3; ++k) {
        double c[4] = {0.0, 0.0, radii[k], 0.0};
        if ((st = nt_add_surface(m, NT_CZ, c, NT_BC_NONE, &sid[6 + k])) != NT_OK) return fail("cz", st);
    }
    const double xs[4][2] = {{0.60, 0.12}, {0.0, 0.0}, {0.30, 0.003}, {1.20, 0.02}};
    for (int k = 0; k < 4; ++k)
        if ((st = nt_add_material(m, xs[k][0], xs[k][1], &mat[k])) != NT_OK) return fail("material", st);
    if ((st = nt_add_csg_universe(m, &root)) != NT_OK) return fail("root", st);
    if ((st = nt_add_csg_universe(m, &pin)) != NT_OK) return fail("pin", st);
    const int32_t box[6] = {sid[0] + 1, -(sid[1] + 1), sid[2] + 1, -(sid[3] + 1), sid[4] + 1, -(sid[5] + 1)};
    if ((st = nt_add_cell(m, root, box, 6, NT_FILL_UNIVERSE, pin, NULL, &cell)) != NT_OK) return fail("box cell", st);
    for (int k = 0; k < 4; ++k) {
        int32_t hs[2];
        int32_t n = 0;
        if (k > 0) hs[n++] = sid[6 + k - 1] + 1;
        if (k < 3) hs[n++] = -(sid[6 + k] + 1);
        if ((st = nt_add_cell(m, pin, hs, n, NT_FILL_MATERIAL, mat[k], NULL, &cell)) != NT_OK) return fail("pin cell", st);
    }
    if ((st = nt_set_root(m, root)) != NT_OK) return fail("root", st);
    /* error path: a material with sigma_a > sigma_t is rejected at finalize (NT_E_GEOMETRY) */
    nt_build_opts o;
    nt_build_opts_default(&o);
    o.device = -1;
    if ((st = nt_finalize(m, &o)) != NT_OK) return fail("finalize", st);
    nt_model_info inf;
    memset(&inf, 0, sizeof(inf));
    if ((st = nt_model_info_get(m, &inf)) != NT_OK) return fail("info", st);
    printf("\"n_surfaces\": %d, \"n_cells\": %d, \"n_material_cells\": %d, \"max_depth\": %d, "
           "\"rect_specialisable\": %d, \"out_len\": %lld, ", inf.n_surfaces, inf.n_cells, inf.n_material_cells,
           inf.max_depth, inf.rect_specialisable, (long long)inf.out_len);
    /* order errors: a builder call after finalize; tracking a host-only model */
    double c[4] = {1.0, 0, 0, 0};
    st = nt_add_surface(m, NT_PX, c, NT_BC_NONE, &id);
    printf("\"add_after_finalize\": %d, ", (int)st);
    nt_run run;
    memset(&run, 0, sizeof(run));
    run.n = 10;
    nt_outputs out;
    memset(&out, 0, sizeof(out));
    double dummy[64];
    out.out = dummy;
    st = nt_track(m, &run, &out, NULL);
    printf("\"track_host_only\": %d, \"track_host_only_msg\": \"%s\", ", (int)st, nt_last_error());
    nt_model_destroy(m);

    /* argument errors: an unknown surface kind, a bad material */
    nt_model* m2 = NULL;
    nt_model_create(&m2);
    st = nt_add_material(m2, 0.5, 0.9, &id);
    printf("\"bad_material\": %d, ", (int)st);
    st = nt_add_surface(m2, (nt_surface_kind)42, c, NT_BC_NONE, &id);
    printf("\"bad_kind\": %d, ", (int)st);
    int32_t u2, c2;
    nt_add_csg_universe(m2, &u2);
    nt_add_cell(m2, u2, NULL, 0, NT_FILL_MATERIAL, 0, NULL, &c2);   /* all of space, the bad material */
    nt_set_root(m2, u2);
    st = nt_finalize(m2, &o);
    printf("\"bad_material_finalize\": %d", (int)st);
    nt_model_destroy(m2);
    printf("}\n");
    return 0;
}
