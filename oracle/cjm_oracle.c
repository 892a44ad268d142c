/*
 * cjm_oracle.c -- plain, slow, obviously-correct CPU oracle of the
 * Chebyshev-Jacobi method (CJM) of arXiv 1705.00103.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_1705_00103_b200/, include/, the CUDA library) may include, link,
 * import or call this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may use it.  It shares no
 * source, header, table or constant generator with the CUDA path.
 *
 * Citation keys: P:L = PAPER.md line L (section / equation named beside it),
 * S:L = SPEC.md line L, "DESIGN R#" = reading number
 * (where the paper is silent, garbled or ambiguous).
 *
 * What it computes, in the paper's order:
 *   1. spectral bounds kappa_min/kappa_max        P:100-106 (Eq. kmkM9p),
 *                                                 P:126-134 (17-pt), 5-pt
 *                                                 classical
 *   2. cycle length M (Chebyshev degree)          P:75-80 "transformation of
 *                                                 the zeros of a Chebyshev
 *                                                 polynomial ... depends on
 *                                                 the tolerance"
 *   3. weights = transformed Chebyshev zeros
 *      applied in a stable order                  DESIGN R3 (paper silent)
 *   4. weighted Jacobi sweeps                     P:73-74 "a weighted classical
 *      u_{n+1} = u_n + w_n D^-1 (b - A u_n)       Jacobi method with strictly
 *                                                 different weights at each
 *                                                 iteration"
 *      with the 5-, 9-, 17-point Laplacians       P:95-99 (Eq. 9-points),
 *                                                 P:118-125 (Eq. 17-points),
 *                                                 P:342-349 (tab:ste2 Cartesian)
 *   5. residual norm at cycle boundaries,         P:459-460 "until reaching a
 *      stop when ||r||_2 <= tol ||r_0||_2         prescribed tolerance";
 *                                                 DESIGN R4
 *   option: 17-point outer ghost ring by odd     P:126-134 (the closed-form
 *      reflection (oracle_odd_closure)            kappa_min^(17) is exact for
 *                                                 it); DESIGN R12
 *
 * Grid convention (DESIGN R1): nx, ny = interior unknowns; the paper's
 * N_x = nx+1, N_y = ny+1 mesh intervals; node (i,j), 1<=i<=nx, 1<=j<=ny; r
 * ghost rings (r=1 for 5/9-pt, r=2 for 17-pt) hold Dirichlet data and are
 * never written.  u is stored row-major with its ghosts: element (i,j) at
 * u[(j-1+r)*ldu + (i-1+r)].  b and g are interior only: (i,j) at
 * b[(j-1)*ldb + (i-1)].
 *
 * Floating point: IEEE fp64 (the paper computes in double precision,
 * P:265-267).  Compiled with -ffp-contract=off; every fused multiply-add is an
 * explicit fma().  The per-point arithmetic is written out below in one fixed
 * association (DESIGN R6) so that a GPU sweep following the same association
 * is bitwise identical.
 *
 * Pins (tests/test_oracle_*.py, all -m "not gpu"): dense eigenvalues of
 * D^-1 A (kappa), Chebyshev T_P product identity and equioscillation
 * (weights), SPEC's worked example M=6, Lebedev-Finogenov theta_8
 * (ordering), dense D^-1(b-Au) and dense matrix polynomial (sweep, cycle),
 * direct sparse solve + manufactured-solution orders (stencils, solve),
 * Fig. 1 golden coefficients.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_OK = 0, OR_INVALID = 1, OR_NOT_CONVERGED = 3, OR_DIVERGED = 4,
       OR_STAGNATED = 5, OR_OOM = 8 };

/* Stencil reach: 5- and 9-point use the 3x3 footprint, the 17-point the 5x5
 * footprint (tab:ste1). */
int oracle_reach(int stencil)
{
    if (stencil == 5 || stencil == 9) return 1;
    if (stencil == 17) return 2;
    return 0;
}

static double sin2(double a) { double s = sin(a); return s * s; }

/* Step 1: closed-form spectral bounds of D^-1 A (DESIGN R1: N = unknowns+1).
 *  9-pt: P:102-104  kmin = 4/5[s2(pi/2Nx)+s2(pi/2Ny)]
 *                        + 1/5[s2(pi/2Nx+pi/2Ny)+s2(pi/2Nx-pi/2Ny)], kmax = 8/5
 * 17-pt: P:128-133  kmin = -4/75[s2(pi/Nx)+s2(pi/Ny)] + 64/75[s2(pi/2Nx)+s2(pi/2Ny)]
 *                        - 1/75[s2(pi/Nx+pi/Ny)+s2(pi/Nx-pi/Ny)]
 *                        + 16/75[s2(pi/2Nx+pi/2Ny)+s2(pi/2Nx-pi/2Ny)], kmax = 128/75
 *                   (braces at P:131-132 garbled; DESIGN R2)
 *  5-pt: classical (not printed): kmin = s2(pi/2Nx)+s2(pi/2Ny), kmax = 2 */
int oracle_bounds(int stencil, int nx, int ny, double *kmin, double *kmax)
{
    if (nx < 1 || ny < 1) return OR_INVALID;
    double Nx = (double)nx + 1.0, Ny = (double)ny + 1.0;
    double hx = M_PI / (2.0 * Nx), hy = M_PI / (2.0 * Ny);   /* pi/2N */
    double fx = M_PI / Nx, fy = M_PI / Ny;                    /* pi/N  */
    if (stencil == 5) {
        *kmin = sin2(hx) + sin2(hy);
        *kmax = 2.0;
    } else if (stencil == 9) {
        *kmin = (4.0 / 5.0) * (sin2(hx) + sin2(hy))
              + (1.0 / 5.0) * (sin2(hx + hy) + sin2(hx - hy));
        *kmax = 8.0 / 5.0;
    } else if (stencil == 17) {
        *kmin = -(4.0 / 75.0) * (sin2(fx) + sin2(fy))
              + (64.0 / 75.0) * (sin2(hx) + sin2(hy))
              - (1.0 / 75.0) * (sin2(fx + fy) + sin2(fx - fy))
              + (16.0 / 75.0) * (sin2(hx + hy) + sin2(hx - hy));
        *kmax = 128.0 / 75.0;
    } else {
        return OR_INVALID;
    }
    return OR_OK;
}

/* Step 2a: minimal Chebyshev degree M with 1/T_M(mu) <= tol, mu =
 * (kmax+kmin)/(kmax-kmin):  M = ceil(acosh(1/tol) / acosh(mu)).
 * acosh(mu) is evaluated as log1p(x + sqrt(x(2+x))), x = 2 kmin/(kmax-kmin),
 * which is the same number without the cancellation of mu - 1 (DESIGN R5). */
long oracle_m_min(double kmin, double kmax, double tol)
{
    double x = 2.0 * kmin / (kmax - kmin);
    double acosh_mu = log1p(x + sqrt(x * (2.0 + x)));
    double m = ceil(acosh(1.0 / tol) / acosh_mu);
    if (m < 1.0) m = 1.0;
    return (long)m;
}

/* Step 2b: cycle length P = the smallest 2^a 3^b >= M (DESIGN R3: the stable
 * ordering below exists for these lengths). */
long oracle_cycle_len(long m_min, int *a_out, int *b_out)
{
    long best = -1; int ba = 0, bb = 0;
    long p2 = 1;
    for (int a = 0; a < 62; a++) {
        long v = p2;
        for (int b = 0; b < 40; b++) {
            if (v >= m_min) {
                if (best < 0 || v < best) { best = v; ba = a; bb = b; }
                break;
            }
            v *= 3;
        }
        if (p2 >= m_min) break;
        p2 *= 2;
    }
    *a_out = ba; *b_out = bb;
    return best;
}

/* Step 2b': the power-of-two cycle of the classical Lebedev-Finogenov
 * ordering (order option LEBEDEV2, DESIGN R3): P = the smallest 2^a >= M. */
long oracle_cycle_len_pow2(long m_min, int *a_out)
{
    long p = 1;
    int a = 0;
    while (p < m_min) { p *= 2; a++; }
    *a_out = a;
    return p;
}

/* Step 3a: order in which the P Chebyshev zeros are applied (DESIGN R3).
 * The paper does not state an order; this is the Lebedev-Finogenov
 * recursion generalised to P = 2^a 3^b.  Start from the list [1] with m = 1;
 * for each factor f of (3 repeated b times, then 2 repeated a times) replace
 * every entry t by (t, 4m - t) when f = 2, by (t, 4m - t, 4m + t) when f = 3,
 * then m <- f m.  The result is a permutation of the odd numbers 1..2P-1;
 * entry k is the index t of the zero cos(t pi / 2P) used at sweep k. */
int oracle_ordering(int a, int b, long *t)
{
    long len = 1, m = 1;
    t[0] = 1;
    for (int step = 0; step < a + b; step++) {
        int f = (step < b) ? 3 : 2;
        /* expand in place from the back so each t[k] is read before it is
         * overwritten */
        for (long k = len - 1; k >= 0; k--) {
            long tk = t[k];
            if (f == 2) {
                t[2 * k] = tk;
                t[2 * k + 1] = 4 * m - tk;
            } else {
                t[3 * k] = tk;
                t[3 * k + 1] = 4 * m - tk;
                t[3 * k + 2] = 4 * m + tk;
            }
        }
        len *= f;
        m *= f;
    }
    return OR_OK;
}

/* Step 3b: the weights, reciprocals of the Chebyshev zeros mapped onto
 * [kmin, kmax]:
 *   w = 2 / [(kmax+kmin) - (kmax-kmin) cos(t pi / 2P)]
 *     = 1 / [kmin + (kmax-kmin) sin^2(t pi / 4P)]        (half-angle identity)
 * evaluated in the sin^2 form, which has no cancellation for the largest
 * weights (DESIGN R5). */
void oracle_weights(double kmin, double kmax, long P, const long *t, double *w)
{
    for (long k = 0; k < P; k++) {
        double theta = (M_PI * (double)t[k]) / (4.0 * (double)P);
        double s = sin(theta);
        w[k] = 1.0 / (kmin + (kmax - kmin) * (s * s));
    }
}

/* D^-1 b: g = (h^2 / c_C) b, c_C = centre coefficient of h^2 Delta_h:
 * -4 (tab:ste2), -20/6 (Eq. 9-points), -300/72 (Eq. 17-points). */
double oracle_gscale(int stencil, double h)
{
    if (stencil == 5) return -(h * h) * 0.25;
    if (stencil == 9) return -(h * h) * 0.3;
    if (stencil == 17) return -(h * h) * (72.0 / 300.0);
    return 0.0;
}

void oracle_rhs_to_g(int stencil, int nx, int ny, double h,
                     const double *b, long ldb, double *g, long ldg)
{
    double gs = oracle_gscale(stencil, h);
    for (int j = 0; j < ny; j++)
        for (int i = 0; i < nx; i++)
            g[(long)j * ldg + i] = gs * b[(long)j * ldb + i];
}

/* The Jacobi correction at one node: d = D^-1 (b - A u) at (i,j)
 *   = g + sum_{k != C} a_k u_k - u_C,   a_k = -c_k / c_C,
 * with the neighbour coefficients of P:95-99 / P:118-125 / tab:ste2 divided
 * by the centre one:
 *   5-pt : a(axis) = 1/4
 *   9-pt : a(axis) = 4/20 = 0.2,  a(diag) = 1/20 = 0.05
 *  17-pt : a(axis,1) = 64/300, a(axis,2) = -4/300,
 *          a(diag,1) = 16/300, a(diag,2) = -1/300
 * Association (DESIGN R6), W/E = x-1/x+1, S/N = y-1/y+1, suffix 2 = distance 2:
 *   S1 = (uW + uE) + (uS + uN)
 *   S2 = (uSW + uSE) + (uNW + uNE)                       [9-pt]
 *   S2 = (uW2 + uE2) + (uS2 + uN2)                        [17-pt]
 *   S3 = (uSW + uSE) + (uNW + uNE)                        [17-pt]
 *   S4 = (uSW2 + uSE2) + (uNW2 + uNE2)                    [17-pt]
 *   J  = fma(a1, S1, fma(a2, S2, ... g))  innermost = highest S index
 *   d  = J - uC                                                            */
static inline double delta_at(int stencil, const double *u, long ldu,
                              long c /* index of (i,j) in u */, double g)
{
    double uC = u[c];
    double uW = u[c - 1], uE = u[c + 1];
    double uS = u[c - ldu], uN = u[c + ldu];
    double S1 = (uW + uE) + (uS + uN);
    double J;
    if (stencil == 5) {
        J = fma(0.25, S1, g);
    } else if (stencil == 9) {
        double uSW = u[c - ldu - 1], uSE = u[c - ldu + 1];
        double uNW = u[c + ldu - 1], uNE = u[c + ldu + 1];
        double S2 = (uSW + uSE) + (uNW + uNE);
        J = fma(0.2, S1, fma(0.05, S2, g));
    } else {
        double uW2 = u[c - 2], uE2 = u[c + 2];
        double uS2 = u[c - 2 * ldu], uN2 = u[c + 2 * ldu];
        double uSW = u[c - ldu - 1], uSE = u[c - ldu + 1];
        double uNW = u[c + ldu - 1], uNE = u[c + ldu + 1];
        double uSW2 = u[c - 2 * ldu - 2], uSE2 = u[c - 2 * ldu + 2];
        double uNW2 = u[c + 2 * ldu - 2], uNE2 = u[c + 2 * ldu + 2];
        double S2 = (uW2 + uE2) + (uS2 + uN2);
        double S3 = (uSW + uSE) + (uNW + uNE);
        double S4 = (uSW2 + uSE2) + (uNW2 + uNE2);
        J = fma(64.0 / 300.0, S1,
            fma(-4.0 / 300.0, S2,
            fma(16.0 / 300.0, S3,
            fma(-1.0 / 300.0, S4, g))));
    }
    return J - uC;
}

/* Step 4: one weighted Jacobi sweep, double buffered (Jacobi, not
 * Gauss-Seidel: every output reads only u_in):
 *   out(i,j) = u(i,j) + w d(i,j)   evaluated as fma(w, d, uC).
 * Only the interior of `out` is written; its ghosts must already hold the
 * Dirichlet data. */
void oracle_sweep(int stencil, int nx, int ny, const double *u, long ldu,
                  const double *g, long ldg, double w, double *out, long ldo)
{
    int r = oracle_reach(stencil);
    #pragma omp parallel for schedule(static)
    for (int j = 1; j <= ny; j++) {
        for (int i = 1; i <= nx; i++) {
            long c = (long)(j - 1 + r) * ldu + (i - 1 + r);
            long co = (long)(j - 1 + r) * ldo + (i - 1 + r);
            double d = delta_at(stencil, u, ldu, c, g[(long)(j - 1) * ldg + (i - 1)]);
            out[co] = fma(w, d, u[c]);
        }
    }
}

/* Step 5 (quantity): sum of d^2 and max |d| over the interior, d = D^-1 r.
 * Sum order is fixed: along each row in increasing x, then over rows in
 * increasing y, so the result does not depend on the thread count. */
void oracle_delta_norms(int stencil, int nx, int ny, const double *u, long ldu,
                        const double *g, long ldg, double *sumsq, double *maxabs)
{
    int r = oracle_reach(stencil);
    double *rs = (double *)malloc(sizeof(double) * (size_t)ny * 2);
    #pragma omp parallel for schedule(static)
    for (int j = 1; j <= ny; j++) {
        double s = 0.0, m = 0.0;
        for (int i = 1; i <= nx; i++) {
            long c = (long)(j - 1 + r) * ldu + (i - 1 + r);
            double d = delta_at(stencil, u, ldu, c, g[(long)(j - 1) * ldg + (i - 1)]);
            s = s + d * d;
            double ad = fabs(d);
            if (ad > m || ad != ad) m = ad;
        }
        rs[2 * (j - 1)] = s;
        rs[2 * (j - 1) + 1] = m;
    }
    double s = 0.0, m = 0.0;
    for (int j = 0; j < ny; j++) {
        s = s + rs[2 * j];
        if (rs[2 * j + 1] > m || rs[2 * j + 1] != rs[2 * j + 1]) m = rs[2 * j + 1];
    }
    free(rs);
    *sumsq = s;
    *maxabs = m;
}

/* Residual r = b - Delta_h u in PDE units: ||r|| = ||d|| / |gscale|
 * (D = c_C / h^2 is a scalar, so r = D d). */
void oracle_residual(int stencil, int nx, int ny, double h,
                     const double *b, long ldb, const double *u, long ldu,
                     double *l2, double *linf)
{
    double *g = (double *)malloc(sizeof(double) * (size_t)nx * ny);
    oracle_rhs_to_g(stencil, nx, ny, h, b, ldb, g, nx);
    double s, m;
    oracle_delta_norms(stencil, nx, ny, u, ldu, g, nx, &s, &m);
    double sc = fabs(oracle_gscale(stencil, h));
    *l2 = sqrt(s) / sc;
    *linf = m / sc;
    free(g);
}

/* 17-point closure option (NEXT-4; DESIGN R12): the outer ghost ring by odd
 * reflection through the boundary instead of given data.  With homogeneous
 * Dirichlet data the 17-point operator then is the odd extension whose
 * smallest eigenvalue the closed form kappa_min^(17) of P:126-134 gives
 * EXACTLY (SURVEY [V2]); with data u_b on the boundary nodes the reflection
 * is affine, u(mirror of i) = 2 u_b - u(i), exact for fields linear across
 * the boundary.  0-based interior (i, j), boundary nodes i = -1, nx and
 * j = -1, ny, outer ring i = -2, nx+1 and j = -2, ny+1; u has r = 2 ghost
 * rings.  Columns first (rows -1..ny), then rows (every column, so the
 * corners of the outer ring reflect the reflected columns):
 *   u(-2, j) = 2 u(-1, j) - u(0, j),   u(nx+1, j) = 2 u(nx, j) - u(nx-1, j)
 *   u(i, -2) = 2 u(i, -1) - u(i, 0),   u(i, ny+1) = 2 u(i, ny) - u(i, ny-1)
 * each as (2.0 * a) - b (2a exact, one rounding). */
void oracle_odd_closure(int nx, int ny, double *u, long ldu)
{
#define U_(i, j) u[(long)((j) + 2) * ldu + ((i) + 2)]
    for (int j = -1; j <= ny; j++) {
        U_(-2, j) = 2.0 * U_(-1, j) - U_(0, j);
        U_(nx + 1, j) = 2.0 * U_(nx, j) - U_(nx - 1, j);
    }
    for (int i = -2; i <= nx + 1; i++) {
        U_(i, -2) = 2.0 * U_(i, -1) - U_(i, 0);
        U_(i, ny + 1) = 2.0 * U_(i, ny) - U_(i, ny - 1);
    }
#undef U_
}

/* `count` consecutive sweeps of the schedule (weight w[(first + k) mod P] at
 * sweep k), double buffered exactly as in oracle_solve; u is overwritten with
 * the result.  Used for fixed segments of a solve at sizes where the whole
 * solve would take the oracle too long. */
int oracle_sweeps(int stencil, int nx, int ny, double *u, long ldu,
                  const double *g, long ldg, const double *w, long P,
                  long first, long count, int closure)
{
    int r = oracle_reach(stencil);
    if (closure && stencil != 17) return OR_INVALID;
    long rows = ny + 2 * r;
    double *v = (double *)malloc(sizeof(double) * (size_t)rows * ldu);
    if (!v) return OR_OOM;
    memcpy(v, u, sizeof(double) * (size_t)rows * ldu);
    double *cur = u, *nxt = v;
    for (long k = 0; k < count; k++) {
        if (closure) oracle_odd_closure(nx, ny, cur, ldu);
        oracle_sweep(stencil, nx, ny, cur, ldu, g, ldg, w[(first + k) % P], nxt, ldu);
        double *tmp = cur; cur = nxt; nxt = tmp;
    }
    if (cur != u)
        memcpy(u, cur, sizeof(double) * (size_t)rows * ldu);
    free(v);
    return OR_OK;
}

typedef struct {
    long long iterations;
    int cycles;
    int status;
    long long cycle_len, m_min;
    double kappa_min, kappa_max;
    double r0_l2, r0_linf, r_l2, r_linf;
} oracle_report;

/* The whole method, step by step:
 *   bounds -> M -> P, ordering, weights -> rho0 = ||r(u0)||_2 ->
 *   repeat cycles of P sweeps (weight k at sweep k of the cycle), after each
 *   cycle rho = ||r(u)||_2 and stop when rho <= tol rho0 (DESIGN R4).
 * Failure modes: non-finite rho -> DIVERGED; rho > rho_prev/2
 * -> STAGNATED (fp64 floor); max_cycles reached -> NOT_CONVERGED.  u then
 * holds the last cycle-boundary iterate.
 * weights_override (may be NULL): run these P weights instead (tests only:
 * e.g. another ordering of the same set).
 * closure = 1 (17-point only): the outer ghost ring by odd reflection,
 * recomputed from the iterate before every sweep and every residual. */
int oracle_solve(int stencil, int nx, int ny, double h, double tol,
                 int max_cycles, const double *b, long ldb, double *u, long ldu,
                 const double *weights_override, long override_len,
                 oracle_report *rep, int closure)
{
    memset(rep, 0, sizeof(*rep));
    int r = oracle_reach(stencil);
    if (!r || nx < 4 || ny < 4 || !(h > 0.0) || !(tol > 0.0 && tol < 1.0)
        || max_cycles < 1 || (closure && stencil != 17))
        return rep->status = OR_INVALID;

    double kmin, kmax;
    oracle_bounds(stencil, nx, ny, &kmin, &kmax);
    long m = oracle_m_min(kmin, kmax, tol);
    int a, bb;
    long P = oracle_cycle_len(m, &a, &bb);
    rep->kappa_min = kmin; rep->kappa_max = kmax;
    rep->m_min = m; rep->cycle_len = P;

    double *w = (double *)malloc(sizeof(double) * (size_t)P);
    long *t = (long *)malloc(sizeof(long) * (size_t)P);
    if (weights_override) {
        P = override_len;
        rep->cycle_len = P;
        w = (double *)realloc(w, sizeof(double) * (size_t)P);
        memcpy(w, weights_override, sizeof(double) * (size_t)P);
    } else {
        oracle_ordering(a, bb, t);
        oracle_weights(kmin, kmax, P, t, w);
    }
    free(t);

    long ldg = nx;
    double *g = (double *)malloc(sizeof(double) * (size_t)nx * ny);
    oracle_rhs_to_g(stencil, nx, ny, h, b, ldb, g, ldg);

    /* second buffer, ghosts copied from u (never written afterwards) */
    long rows = ny + 2 * r;
    double *v = (double *)malloc(sizeof(double) * (size_t)rows * ldu);
    if (!w || !g || !v) { free(w); free(g); free(v); return rep->status = OR_OOM; }
    memcpy(v, u, sizeof(double) * (size_t)rows * ldu);

    double sc = fabs(oracle_gscale(stencil, h));
    double s, mx;
    if (closure) oracle_odd_closure(nx, ny, u, ldu);
    oracle_delta_norms(stencil, nx, ny, u, ldu, g, ldg, &s, &mx);
    rep->r0_l2 = sqrt(s) / sc;
    rep->r0_linf = mx / sc;
    rep->r_l2 = rep->r0_l2;
    rep->r_linf = rep->r0_linf;
    if (rep->r0_l2 == 0.0) {
        free(w); free(g); free(v);
        return rep->status = OR_OK;
    }

    double *cur = u, *nxt = v;
    double rho_prev = rep->r0_l2;
    int status = OR_NOT_CONVERGED;
    for (int c = 1; c <= max_cycles; c++) {
        for (long k = 0; k < P; k++) {
            if (closure) oracle_odd_closure(nx, ny, cur, ldu);
            oracle_sweep(stencil, nx, ny, cur, ldu, g, ldg, w[k], nxt, ldu);
            double *tmp = cur; cur = nxt; nxt = tmp;
        }
        rep->iterations += P;
        rep->cycles = c;
        if (closure) oracle_odd_closure(nx, ny, cur, ldu);
        oracle_delta_norms(stencil, nx, ny, cur, ldu, g, ldg, &s, &mx);
        double rho = sqrt(s) / sc;
        rep->r_l2 = rho;
        rep->r_linf = mx / sc;
        if (!isfinite(rho)) { status = OR_DIVERGED; break; }
        if (rho <= tol * rep->r0_l2) { status = OR_OK; break; }
        if (rho > 0.5 * rho_prev) { status = OR_STAGNATED; break; }
        rho_prev = rho;
    }
    if (cur != u)
        memcpy(u, cur, sizeof(double) * (size_t)rows * ldu);
    free(w); free(g); free(v);
    return rep->status = status;
}

/* ---------------------------------------------------------------------------
 * Generic 5-point masks (NEXT-4, tab:ste1 upper part, tab:ste2):
 * per-node coefficients c_W, c_E, c_S, c_N, c_C (PDE units, row-major
 * ny x nx, pitch ldc) -- "both the central node ... and each of its neighbors
 * ... can have different numerical factors".  The Jacobi
 * correction of node (i,j) (DESIGN R10, one fixed association):
 *   a_k = -c_k / c_C,  g = b / c_C,
 *   J = fma(a_W, uW, fma(a_E, uE, fma(a_S, uS, fma(a_N, uN, g)))),
 *   d = J - uC,   u' = fma(w, d, uC),   r = c_C d.
 * ------------------------------------------------------------------------- */
void oracle_mask_sweep(int nx, int ny, const double *u, long ldu, const double *cW,
                       const double *cE, const double *cS, const double *cN, const double *cC,
                       long ldc, const double *b, long ldb, double w, double *out, long ldo)
{
    #pragma omp parallel for schedule(static)
    for (int j = 1; j <= ny; j++) {
        for (int i = 1; i <= nx; i++) {
            long c = (long)j * ldu + i;          /* one ghost ring */
            long k = (long)(j - 1) * ldc + (i - 1);
            long kb = (long)(j - 1) * ldb + (i - 1);
            double cc = cC[k];
            double aW = -cW[k] / cc, aE = -cE[k] / cc, aS = -cS[k] / cc, aN = -cN[k] / cc;
            double g = b[kb] / cc;
            double J = fma(aW, u[c - 1], fma(aE, u[c + 1], fma(aS, u[c - ldu], fma(aN, u[c + ldu], g))));
            out[(long)j * ldo + i] = fma(w, J - u[c], u[c]);
        }
    }
}

/* ||r||_2, ||r||_inf with r = c_C d (the residual in PDE units). */
void oracle_mask_residual(int nx, int ny, const double *u, long ldu, const double *cW,
                          const double *cE, const double *cS, const double *cN,
                          const double *cC, long ldc, const double *b, long ldb,
                          double *l2, double *linf)
{
    double *rs = (double *)malloc(sizeof(double) * (size_t)ny * 2);
    #pragma omp parallel for schedule(static)
    for (int j = 1; j <= ny; j++) {
        double s = 0.0, m = 0.0;
        for (int i = 1; i <= nx; i++) {
            long k = (long)(j - 1) * ldc + (i - 1);
            long c = (long)j * ldu + i;
            double cc = cC[k];
            double aW = -cW[k] / cc, aE = -cE[k] / cc, aS = -cS[k] / cc, aN = -cN[k] / cc;
            double g = b[(long)(j - 1) * ldb + (i - 1)] / cc;
            double J = fma(aW, u[c - 1], fma(aE, u[c + 1], fma(aS, u[c - ldu], fma(aN, u[c + ldu], g))));
            double r = cc * (J - u[c]);
            s = s + r * r;
            double ar = fabs(r);
            if (ar > m || ar != ar) m = ar;
        }
        rs[2 * (j - 1)] = s;
        rs[2 * (j - 1) + 1] = m;
    }
    double s = 0.0, m = 0.0;
    for (int j = 0; j < ny; j++) {
        s = s + rs[2 * j];
        if (rs[2 * j + 1] > m || rs[2 * j + 1] != rs[2 * j + 1]) m = rs[2 * j + 1];
    }
    free(rs);
    *l2 = sqrt(s);
    *linf = m;
}

/* The CJM with a generic mask and caller-supplied spectral bounds (there is
 * no closed form off the Cartesian grid): M, P, ordering and
 * weights exactly as for the Cartesian stencils, stop as in oracle_solve. */
int oracle_mask_solve(int nx, int ny, const double *cW, const double *cE, const double *cS,
                      const double *cN, const double *cC, long ldc, const double *b, long ldb,
                      double kmin, double kmax, double tol, int max_cycles,
                      double *u, long ldu, oracle_report *rep)
{
    memset(rep, 0, sizeof(*rep));
    if (nx < 1 || ny < 1 || !(kmin > 0.0 && kmax > kmin) || !(tol > 0.0 && tol < 1.0))
        return rep->status = OR_INVALID;
    long m = oracle_m_min(kmin, kmax, tol);
    int a, bb;
    long P = oracle_cycle_len(m, &a, &bb);
    rep->kappa_min = kmin; rep->kappa_max = kmax; rep->m_min = m; rep->cycle_len = P;
    long *t = (long *)malloc(sizeof(long) * (size_t)P);
    double *w = (double *)malloc(sizeof(double) * (size_t)P);
    oracle_ordering(a, bb, t);
    oracle_weights(kmin, kmax, P, t, w);
    free(t);
    long rows = ny + 2;
    double *v = (double *)malloc(sizeof(double) * (size_t)rows * ldu);
    memcpy(v, u, sizeof(double) * (size_t)rows * ldu);
    double l2, li;
    oracle_mask_residual(nx, ny, u, ldu, cW, cE, cS, cN, cC, ldc, b, ldb, &l2, &li);
    rep->r0_l2 = rep->r_l2 = l2;
    rep->r0_linf = rep->r_linf = li;
    int status = OR_NOT_CONVERGED;
    if (l2 == 0.0) status = OR_OK;
    double *cur = u, *nxt = v;
    double rho_prev = l2;
    for (int c = 1; status == OR_NOT_CONVERGED && c <= max_cycles; c++) {
        for (long k = 0; k < P; k++) {
            oracle_mask_sweep(nx, ny, cur, ldu, cW, cE, cS, cN, cC, ldc, b, ldb, w[k], nxt, ldu);
            double *tmp = cur; cur = nxt; nxt = tmp;
        }
        rep->iterations += P;
        rep->cycles = c;
        oracle_mask_residual(nx, ny, cur, ldu, cW, cE, cS, cN, cC, ldc, b, ldb, &l2, &li);
        rep->r_l2 = l2;
        rep->r_linf = li;
        if (!isfinite(l2)) { status = OR_DIVERGED; break; }
        if (l2 <= tol * rep->r0_l2) { status = OR_OK; break; }
        if (l2 > 0.5 * rho_prev) { status = OR_STAGNATED; break; }
        rho_prev = l2;
    }
    if (cur != u) memcpy(u, cur, sizeof(double) * (size_t)rows * ldu);
    free(v); free(w);
    return rep->status = status;
}

/* ---------------------------------------------------------------------------
 * Generic (2m+1) x (2m+1) masks, m = 1 or 2 (NEXT-4, tab:ste1):
 * "both the central node ... and each of its (at most) 24 neighbors spanned
 * by the discretization of the Laplacian can have different numerical
 * factors" which "may change as a function of the position of the central
 * node".  m = 1 is the upper part of tab:ste1 (up to 9 points), m = 2 the
 * most generic case (lower part, up to 25 points).  c[q] (q = (dy+m)(2m+1) +
 * (dx+m), dx, dy in -m..m; x = first index, y = second) is the per-node
 * coefficient of neighbour (i+dx, j+dy), row-major ny x nx with pitch ldc, or
 * NULL for a neighbour that is absent everywhere; q_C = m(2m+1)+m is the
 * centre.  u has m ghost rings: node (i,j) at u[(j-1+m) ldu + (i-1+m)].
 * The Jacobi correction (DESIGN R11, one fixed association):
 *   a_q = -c_q / c_C,  g = b / c_C,
 *   J = fma(a_0, u_0, fma(a_1, u_1, ... fma(a_{Q-1}, u_{Q-1}, g)))  over the
 *       present neighbours in increasing q (the innermost is the largest q),
 *   d = J - uC,   u' = fma(w, d, uC),   r = c_C d.
 * ------------------------------------------------------------------------- */
static double maskn_d(int m, int i, int j, const double *u, long ldu, const double *const *c,
                      long ldc, const double *b, long ldb, double *cc_out)
{
    int s = 2 * m + 1, qc = m * s + m;
    long k = (long)(j - 1) * ldc + (i - 1);
    double cc = c[qc][k];
    double J = b[(long)(j - 1) * ldb + (i - 1)] / cc;
    for (int q = s * s - 1; q >= 0; q--) {
        if (q == qc || !c[q]) continue;
        int dy = q / s - m, dx = q % s - m;
        double a = -c[q][k] / cc;
        J = fma(a, u[(long)(j - 1 + m + dy) * ldu + (i - 1 + m + dx)], J);
    }
    *cc_out = cc;
    return J - u[(long)(j - 1 + m) * ldu + (i - 1 + m)];
}

void oracle_maskn_sweep(int m, int nx, int ny, const double *u, long ldu, const double *const *c,
                        long ldc, const double *b, long ldb, double w, double *out, long ldo)
{
    #pragma omp parallel for schedule(static)
    for (int j = 1; j <= ny; j++) {
        for (int i = 1; i <= nx; i++) {
            double cc;
            double d = maskn_d(m, i, j, u, ldu, c, ldc, b, ldb, &cc);
            double uc = u[(long)(j - 1 + m) * ldu + (i - 1 + m)];
            out[(long)(j - 1 + m) * ldo + (i - 1 + m)] = fma(w, d, uc);
        }
    }
}

/* ||r||_2, ||r||_inf of r = c_C d; row sums in column order, rows in order. */
void oracle_maskn_residual(int m, int nx, int ny, const double *u, long ldu,
                           const double *const *c, long ldc, const double *b, long ldb,
                           double *l2, double *linf)
{
    double *rs = (double *)malloc(sizeof(double) * (size_t)ny * 2);
    #pragma omp parallel for schedule(static)
    for (int j = 1; j <= ny; j++) {
        double s = 0.0, mx = 0.0;
        for (int i = 1; i <= nx; i++) {
            double cc;
            double d = maskn_d(m, i, j, u, ldu, c, ldc, b, ldb, &cc);
            double r = cc * d;
            s = s + r * r;
            double ar = fabs(r);
            if (ar > mx || ar != ar) mx = ar;
        }
        rs[2 * (j - 1)] = s;
        rs[2 * (j - 1) + 1] = mx;
    }
    double s = 0.0, mx = 0.0;
    for (int j = 0; j < ny; j++) {
        s = s + rs[2 * j];
        if (rs[2 * j + 1] > mx || rs[2 * j + 1] != rs[2 * j + 1]) mx = rs[2 * j + 1];
    }
    free(rs);
    *l2 = sqrt(s);
    *linf = mx;
}

/* The CJM with a generic (2m+1)^2 mask and caller-supplied spectral bounds. */
int oracle_maskn_solve(int m, int nx, int ny, const double *const *c, long ldc, const double *b,
                       long ldb, double kmin, double kmax, double tol, int max_cycles,
                       double *u, long ldu, oracle_report *rep)
{
    memset(rep, 0, sizeof(*rep));
    if (m < 1 || m > 2 || nx < 1 || ny < 1 || !(kmin > 0.0 && kmax > kmin) ||
        !(tol > 0.0 && tol < 1.0))
        return rep->status = OR_INVALID;
    long mm = oracle_m_min(kmin, kmax, tol);
    int a, bb;
    long P = oracle_cycle_len(mm, &a, &bb);
    rep->kappa_min = kmin; rep->kappa_max = kmax; rep->m_min = mm; rep->cycle_len = P;
    long *t = (long *)malloc(sizeof(long) * (size_t)P);
    double *w = (double *)malloc(sizeof(double) * (size_t)P);
    oracle_ordering(a, bb, t);
    oracle_weights(kmin, kmax, P, t, w);
    free(t);
    long rows = ny + 2 * m;
    double *v = (double *)malloc(sizeof(double) * (size_t)rows * ldu);
    memcpy(v, u, sizeof(double) * (size_t)rows * ldu);
    double l2, li;
    oracle_maskn_residual(m, nx, ny, u, ldu, c, ldc, b, ldb, &l2, &li);
    rep->r0_l2 = rep->r_l2 = l2;
    rep->r0_linf = rep->r_linf = li;
    int status = OR_NOT_CONVERGED;
    if (l2 == 0.0) status = OR_OK;
    double *cur = u, *nxt = v;
    double rho_prev = l2;
    for (int cyc = 1; status == OR_NOT_CONVERGED && cyc <= max_cycles; cyc++) {
        for (long k = 0; k < P; k++) {
            oracle_maskn_sweep(m, nx, ny, cur, ldu, c, ldc, b, ldb, w[k], nxt, ldu);
            double *tmp = cur; cur = nxt; nxt = tmp;
        }
        rep->iterations += P;
        rep->cycles = cyc;
        oracle_maskn_residual(m, nx, ny, cur, ldu, c, ldc, b, ldb, &l2, &li);
        rep->r_l2 = l2;
        rep->r_linf = li;
        if (!isfinite(l2)) { status = OR_DIVERGED; break; }
        if (l2 <= tol * rep->r0_l2) { status = OR_OK; break; }
        if (l2 > 0.5 * rho_prev) { status = OR_STAGNATED; break; }
        rho_prev = l2;
    }
    if (cur != u) memcpy(u, cur, sizeof(double) * (size_t)rows * ldu);
    free(v); free(w);
    return rep->status = status;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
