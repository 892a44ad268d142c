/*
 * A plain C client of the C ABI (include/cjm.h), no Python, no torch:
 *   c_abi_demo host      -- host-only entry points (scheduler, slab / halo
 *                           geometry, buffer layout, status strings)
 *   c_abi_demo solve N   -- the paper's test problem on an N x N
 *                           grid solved with cjm_solve_host from host buffers
 *                           (one H2D, one D2H); prints the report
 *                           and the interior field to stdout as hex doubles
 * Output: one JSON object per line (tests/test_c_abi.py reads it).
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cjm.h"

static int host_part(void) {
    double kmin, kmax;
    long long m, P;
    cjm_status s = cjm_schedule(CJM_STENCIL_9, 64, 64, 1e-8, CJM_ORDER_LEBEDEV23, &kmin, &kmax, &m, &P,
                                NULL, NULL, 0);
    if (s != CJM_OK) return 1;
    long long *t = malloc(sizeof(long long) * (size_t)P);
    double *w = malloc(sizeof(double) * (size_t)P);
    s = cjm_schedule(CJM_STENCIL_9, 64, 64, 1e-8, CJM_ORDER_LEBEDEV23, NULL, NULL, NULL, NULL, t, w, P);
    if (s != CJM_OK) return 1;
    printf("{\"kind\": \"schedule\", \"version\": %d, \"kappa_min\": \"%a\", \"kappa_max\": \"%a\", "
           "\"m_min\": %lld, \"P\": %lld, \"t0\": %lld, \"t1\": %lld, \"w0\": \"%a\", \"wlast\": \"%a\"}\n",
           cjm_version(), kmin, kmax, m, P, t[0], t[1], w[0], w[P - 1]);
    /* too small a capacity is an error, not a buffer overrun */
    s = cjm_schedule(CJM_STENCIL_9, 64, 64, 1e-8, CJM_ORDER_LEBEDEV23, NULL, NULL, NULL, NULL, t, w, P - 1);
    printf("{\"kind\": \"capacity\", \"status\": \"%s\"}\n", cjm_status_str(s));
    free(t);
    free(w);
    int y0, nyl;
    cjm_slab(16384, 8, 3, &y0, &nyl);
    cjm_halo_xfer xs[2];
    int nx = 0;
    long long ld = 0;
    s = cjm_halo_xfers(16384, 16384, 4, 8, 3, xs, &nx, &ld);
    long long ld2;
    int col0;
    cjm_buffer_layout(16384, &ld2, &col0);
    printf("{\"kind\": \"geometry\", \"y0\": %d, \"ny_local\": %d, \"nxfers\": %d, \"ld\": %lld, "
           "\"ld_layout\": %lld, \"col0\": %d, \"peer0\": %d, \"send0\": %lld, \"recv0\": %lld, "
           "\"count0\": %lld, \"status\": \"%s\"}\n",
           y0, nyl, nx, ld, ld2, col0, xs[0].peer, xs[0].send_off, xs[0].recv_off, xs[0].count,
           cjm_status_str(s));
    return 0;
}

static int solve_part(int n) {
    /* the paper's test problem: Delta u = -(x^2+y^2) e^{xy}, u = -e^{xy} on
     * the boundary, u0 = 0 inside; h = 1/(n+1) (DESIGN R1, section 4) */
    const int r = 1;
    const double h = 1.0 / (n + 1);
    const long long ldu = n + 2 * r;
    double *u = calloc((size_t)ldu * (n + 2 * r), sizeof(double));
    double *b = malloc(sizeof(double) * (size_t)n * n);
    for (int j = 0; j < n + 2 * r; j++)
        for (int i = 0; i < n + 2 * r; i++) {
            const double x = (i + 1 - r) * h, y = (j + 1 - r) * h;
            const int ghost = i < r || i >= n + r || j < r || j >= n + r;
            u[(long long)j * ldu + i] = ghost ? -exp(x * y) : 0.0;
        }
    for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++) {
            const double x = (i + 1) * h, y = (j + 1) * h;
            b[(long long)j * n + i] = -(x * x + y * y) * exp(x * y);
        }
    /* the inputs exactly as built here (libm's exp), for the oracle */
    printf("{\"kind\": \"inputs\", \"n\": %d, \"h\": \"%a\", \"u0\": [", n, h);
    for (long long k = 0; k < ldu * (n + 2 * r); k++) printf("%s\"%a\"", k ? ", " : "", u[k]);
    printf("], \"b\": [");
    for (long long k = 0; k < (long long)n * n; k++) printf("%s\"%a\"", k ? ", " : "", b[k]);
    printf("]}\n");
    cjm_options opt;
    cjm_default_options(&opt);
    cjm_plan_t plan = NULL;
    cjm_status s = cjm_plan(&plan, CJM_STENCIL_9, n, n, h, CJM_BC_DIRICHLET, 1e-8, &opt);
    if (s != CJM_OK) {
        printf("{\"kind\": \"error\", \"where\": \"cjm_plan\", \"status\": \"%s\", \"msg\": \"%s\"}\n",
               cjm_status_str(s), cjm_last_error());
        return 1;
    }
    cjm_report rep;
    s = cjm_solve_host(plan, b, n, u, ldu, NULL, &rep);
    cjm_plan_destroy(plan);
    printf("{\"kind\": \"solve\", \"status\": \"%s\", \"iterations\": %lld, \"cycles\": %d, "
           "\"r_ratio\": %.6e, \"h2d_bytes\": %.0f, \"d2h_bytes\": %.0f}\n",
           cjm_status_str(s), rep.iterations, rep.cycles, rep.r_l2 / rep.r0_l2, rep.h2d_bytes,
           rep.d2h_bytes);
    printf("{\"kind\": \"field\", \"n\": %d, \"values\": [", n);
    for (int j = 0; j < n; j++)
        for (int i = 0; i < n; i++)
            printf("%s\"%a\"", (i || j) ? ", " : "", u[(long long)(j + r) * ldu + i + r]);
    printf("]}\n");
    free(u);
    free(b);
    return s == CJM_OK ? 0 : 1;
}

int main(int argc, char **argv) {
    if (argc > 1 && strcmp(argv[1], "solve") == 0) return solve_part(argc > 2 ? atoi(argv[2]) : 64);
    return host_part();
}
