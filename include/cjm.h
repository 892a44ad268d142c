/*
 * cjm.h -- C ABI of the B200-native Chebyshev-Jacobi (CJM) solver, the hot
 * path of arXiv 1705.00103 ("Speeding up a few orders of magnitude the Jacobi
 * method: high order Chebyshev-Jacobi over GPUs").
 *
 * Citation keys: P:L = PAPER.md line L (section / equation named beside it);
 * S:L = SPEC.md line L; DESIGN R# = reading
 *
 * The method (section 2.1): a weighted classical Jacobi iteration
 *     u_{n+1} = u_n + w_n D^{-1} (b - A u_n)
 * with a different weight w_n at every sweep, the weights being "a
 * transformation of the zeros of a Chebyshev polynomial" that depends on "the
 * resolution of the mesh, the boundary conditions and the required
 * tolerance", applied cyclically until "reaching a prescribed
 * tolerance".  A = Delta_h is the 5-point (tab:ste2),
 * 9-point alpha=2/3 (Eq. 9-points) or 17-point alpha=2/3
 * (Eq. 17-points) Laplacian on a uniform grid with
 * Dirichlet data.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - nx, ny: interior unknowns (DESIGN R1: the paper's N_x = nx+1 intervals).
 *    Node (i,j), 1 <= i <= nx, 1 <= j <= ny, sits at (i h, j h).
 *  - r = stencil reach: 1 for the 5- and 9-point, 2 for the 17-point
 *    (the paper's 3x3 and 5x5 masks, tab:ste1 / P:403-409).
 *  - u: fp64, row-major, WITH its r ghost rings: (rows_u) x (nx + 2r) values
 *    in rows of pitch ld_u >= nx + 2r doubles; node (i,j) at
 *    u[(j - 1 + r) * ld_u + (i - 1 + r)].  Ghost values are the Dirichlet
 *    data and are never written.  Interior values are the initial guess on
 *    entry and the solution on return.
 *  - rhs: fp64, row-major, interior only: ny x nx values of pitch
 *    ld_rhs >= nx; node (i,j) at rhs[(j-1) * ld_rhs + (i-1)].  rhs is b in
 *    PDE units (Delta u = b, the paper's test problem P:441); read only.
 *  - Multi-GPU (world_size > 1): rank g owns the row slab
 *    [y0, y0 + ny_local) of the global interior rows (cjm_plan_info); u and
 *    rhs are then the LOCAL slab (rows_u = ny_local + 2r, rhs ny_local rows).
 *    Ghost rows that border another rank are filled by the library (halo
 *    exchange of K r rows after every K-fused launch); only
 *    ranks 0 and world_size-1 need real top / bottom data.  external_halo
 *    plans with temporal_k = K > 1 instead take u with H = K r ghost rows and
 *    rhs with H extra rows above and below (the neighbours' rows, refreshed
 *    by the caller): cjm_report.ghost_rows / rhs_ghost_rows say how many.
 *  - Every call returns a cjm_status; no exception crosses the ABI.  On
 *    CJM_ERR_CUDA / CJM_ERR_NCCL, cjm_last_error() gives the message.
 *  - Thread compatibility: a plan may be used by one host thread at a time.
 *  - Device pointers must come from cudaMalloc-class allocations on the
 *    plan's device (e.g. torch CUDA tensors); host pointers may be pageable
 *    or pinned (pinned is faster).
 */
#ifndef CJM_H
#define CJM_H

#ifdef __cplusplus
extern "C" {
#endif

#define CJM_VERSION_MAJOR 0
#define CJM_VERSION_MINOR 1

typedef enum {
    CJM_OK = 0,
    CJM_ERR_INVALID_ARG = 1,   /* bad size / pointer / tol / option */
    CJM_ERR_UNSUPPORTED = 2,   /* e.g. a boundary condition other than Dirichlet */
    CJM_ERR_NOT_CONVERGED = 3, /* max_cycles reached */
    CJM_ERR_DIVERGED = 4,      /* non-finite residual */
    CJM_ERR_STAGNATED = 5,     /* a cycle reduced ||r||_2 by less than 2x (fp64 floor) */
    CJM_ERR_CUDA = 6,
    CJM_ERR_NCCL = 7,
    CJM_ERR_OOM = 8
} cjm_status;

/* The three Laplacians of the paper (value = number of points), and the
 * generic per-node 5-point mask (tab:ste1 / tab:ste2; plans made
 * with cjm_plan_mask only). */
typedef enum {
    CJM_STENCIL_MASK = 1,
    CJM_STENCIL_5 = 5,
    CJM_STENCIL_9 = 9,
    CJM_STENCIL_17 = 17
} cjm_stencil;

/* Only Dirichlet data is covered by the paper's closed-form kappa bounds
 * (S:322).  Any other value -> CJM_ERR_UNSUPPORTED. */
typedef enum { CJM_BC_DIRICHLET = 0 } cjm_bc;

/* Order in which the weights of a cycle are applied (DESIGN R3; the paper is
 * silent: "precalculated ... as a transformation of the zeros").
 * LEBEDEV23 is the stable default: cycle length P = smallest 2^a 3^b >= M_min
 * (<= 5.2% more sweeps than M_min at every config), generalised
 * Lebedev-Finogenov recursion.  LEBEDEV2 is the classical power-of-two case:
 * P = smallest 2^a >= M_min (up to 2x M_min sweeps), the same recursion with
 * factors of 2 only.  ASCENDING is SPEC's order with the 2^a 3^b
 * cycle, unstable in fp64, offered for tests only. */
typedef enum {
    CJM_ORDER_LEBEDEV23 = 0,
    CJM_ORDER_ASCENDING = 1,
    CJM_ORDER_LEBEDEV2 = 2
} cjm_order;

/* CHEBYSHEV = the CJM.  JACOBI = the classical Jacobi baseline the
 * paper compares against (w = 1); its "cycle" is a
 * check interval of jacobi_check sweeps and it has no stagnation test. */
typedef enum { CJM_METHOD_CHEBYSHEV = 0, CJM_METHOD_JACOBI = 1 } cjm_method;

/* Outer ghost ring of the 17-point stencil (reach 2).  DIRICHLET: the
 * caller's data in both rings, never written (the test problem's analytic
 * values; the closed-form kappa_min^(17) is then a lower bound of
 * lambda_min, DESIGN R2).  ODD: the outer ring is set by odd reflection
 * through the boundary, u(mirror) = 2 u_b - u (the boundary ring u_b is the
 * Dirichlet data), recomputed from the iterate before every sweep and every
 * residual: the iteration operator is then the odd extension whose
 * lambda_min the closed form P:126-134 gives exactly (DESIGN R12, SURVEY
 * [V2]). */
typedef enum { CJM_CLOSURE_DIRICHLET = 0, CJM_CLOSURE_ODD = 1 } cjm_closure;

typedef struct {
    int max_cycles;        /* default 8 (Jacobi: default 100000) */
    int order;             /* cjm_order, default CJM_ORDER_LEBEDEV23 */
    int method;            /* cjm_method, default CJM_METHOD_CHEBYSHEV */
    int jacobi_check;      /* Jacobi check interval in sweeps, default 1024 */
    int world_size;        /* default 1 (single GPU) */
    int rank;              /* default 0 */
    const void *nccl_id;   /* 128-byte ncclUniqueId from cjm_get_nccl_id on rank 0,
                              broadcast by the caller; required when world_size > 1
                              (unless external_halo).  With world_size = 1 a non-NULL
                              id makes a ONE-rank communicator: the plan then runs the
                              multi-GPU schedule (NCCL groups, comm-stream overlap,
                              allreduce) on one GPU.  Communicators are cached by
                              (id, world, rank, device): a later plan with the same id
                              reuses the idle communicator without a collective call;
                              every rank must make the same plan calls in the same
                              order, and a second LIVE plan with an id in use is
                              INVALID_ARG (ids are single-use for initialisation). */
    int device;            /* CUDA device ordinal; -1 (default) = current device */
    int external_halo;     /* world_size > 1 only: 1 = no NCCL; the caller moves the
                              halo rows itself between cjm_sweeps calls (rows from
                              cjm_halo_plan) and combines slab-local residuals.
                              cjm_solve / cjm_solve_host then return UNSUPPORTED. */
    /* tuning knobs, 0 = automatic */
    int temporal_k;        /* sweeps fused per kernel launch (temporal blocking,
                              SURVEY NEXT-1), 1..4 (0 = 4 for the 5/9-point and 3 for
                              the 17-point from 4096^2 up, one less below).  Multi-GPU
                              plans keep K and exchange H = K r halo rows per launch
                              (deep halos); K falls back to 1 when a slab is thinner
                              than 2 K r + 1 rows */
    int variant;           /* sweep kernel, both bitwise identical: 7 = warp-tiled
                              (2 columns per lane, 2r+1 rows per TMA ring stage; the
                              default, 17-point up to temporal_k 3); 3 = shared-line
                              levels (the 17-point at temporal_k 4, or tile_w given) */
    int tile_w;            /* variant 3 only: tile columns per CTA, 256 or 512 */
    int ctas_per_sm;       /* resident CTAs per SM of the persistent sweep grid */
    int stages;            /* depth of the TMA ring (stages of 2r+1 rows for variant 7,
                              one row for variant 3) */
    int graph_chunk;       /* sweeps captured per CUDA graph */
    int resident;          /* hot sweeps of grids that fit in the SMs' shared memory run
                              as ONE cooperative launch per cycle with the grid resident
                              in shared memory: 0 = auto (default), 1 = required,
                              -1 = never.  Single GPU only. */
    int band_split;        /* 1: run every hot launch as two boundary-band launches
                              (H rows each) + the interior launch (the multi-GPU
                              overlap schedule) even without NCCL; for tests */
    int warps;             /* variant 7 only: consumer warps per CTA, 4, 5 or 7, or 11
                              (5/9-point at temporal_k 4: one CTA per SM); 0 = the
                              count that keeps the most consumer warps resident per
                              SM */
    int closure;           /* cjm_closure, default DIRICHLET.  ODD: 17-point only,
                              single GPU, one sweep per launch (temporal_k 0 or 1),
                              no resident kernel; else INVALID_ARG.  The caller's
                              outer ring is read but never written (the library
                              reflects into its own buffers). */
    int chunk_rows;        /* warp-tiled kernel, non-reducing launches: every CTA
                              streams a static range of 80% of its share of the
                              (strip, row) units, the last 20% go out in work items of
                              chunk_rows units that the CTAs take from a device counter
                              (dynamic load balancing); 0 = automatic (1/8 of a CTA's
                              share, 16..128), -1 = static ranges only.  The fraction
                              can be overridden with CJM_DYN_PCT (0..100) for tuning */
} cjm_options;

typedef struct {
    long long iterations;  /* sweeps applied to the returned iterate */
    int cycles;            /* completed cycles (checks after r0) */
    int status;            /* cjm_status of the solve */
    long long cycle_len;   /* P (sweeps per cycle) */
    long long m_min;       /* minimal Chebyshev degree M for tol */
    double kappa_min, kappa_max;
    double r0_l2, r0_linf; /* ||b - Delta_h u_0||, PDE units, global */
    double r_l2, r_linf;   /* same for the returned iterate */
    double plan_s;         /* host seconds spent in cjm_plan */
    double solve_s;        /* device seconds of the solve (CUDA events, whole call) */
    double sweep_s;        /* device seconds of the non-check sweeps (CUDA events) */
    long long sweeps_timed;/* number of sweeps inside sweep_s */
    long long kernel_launches; /* kernels of this library launched by the call */
    long long hot_launches;    /* sweep-kernel launches inside sweep_s */
    int temporal_k;            /* sweeps per hot launch (streaming kernels) */
    int resident;              /* 1: hot sweeps ran in the shared-memory-resident kernel */
    int ghost_rows;            /* ghost rows above / below the slab in the caller's u */
    int rhs_ghost_rows;        /* extra rows above / below the slab in the caller's rhs */
    double h2d_bytes, d2h_bytes;  /* host<->device bytes moved by the call */
    double real_error;     /* cjm_solve_ref: max |u - u_ref| of the returned iterate */
    int variant, warps, stages, ctas;  /* launch configuration of the plan's sweep kernel:
                                          variant, consumer warps per CTA, TMA ring
                                          stages, persistent CTAs */
    int comm_nranks;       /* ranks of the plan's NCCL communicator (0: none) */
    int comm_rank;         /* this plan's rank in it (-1: none) */
} cjm_report;

typedef struct cjm_plan_s *cjm_plan_t;

/* Fill *opt with the defaults above. */
void cjm_default_options(cjm_options *opt);

/* Host-only scheduler (no GPU needed): SURVEY section 8(a) rows a1-a4.
 *   kappa bounds (5-pt classical S:252) at
 *   N_x = nx+1, N_y = ny+1 (DESIGN R1); M_min = ceil(acosh(1/tol)/acosh(mu))
 *   (DESIGN R5); P = smallest 2^a 3^b >= M_min (LEBEDEV2: 2^a) and
 *   the application order t_1..t_P (DESIGN R3);
 *   w_k = 1/(kmin + (kmax-kmin) sin^2(t_k pi/4P)).
 * Outputs: kappa_min, kappa_max, m_min, cycle_len (= P) always (nullable);
 * t_out / w_out (nullable) receive P entries if capacity >= P, else
 * CJM_ERR_INVALID_ARG (call once with capacity 0 to learn P).
 * Errors: INVALID_ARG for nx or ny < 4, tol outside (0,1), an
 * unknown stencil or order. */
cjm_status cjm_schedule(int stencil, int nx, int ny, double tol, int order,
                        double *kappa_min, double *kappa_max,
                        long long *m_min, long long *cycle_len,
                        long long *t_out, double *w_out, long long capacity);

/* Build a plan: run the scheduler, pick the launch configuration, allocate
 * the work buffers on the device (two iterate buffers, g = D^-1 b, the
 * weights, reduction scratch, the NCCL communicator when world_size > 1)
 * and copy the weights host->device once.
 *   h: uniform mesh spacing, > 0 and finite.
 * Ownership: the plan owns all its buffers until cjm_plan_destroy.
 * Errors: INVALID_ARG (sizes, h, tol, options; a slab thinner than 2r+1
 * rows), UNSUPPORTED (bc), OOM, CUDA, NCCL.  *out is NULL on error. */
cjm_status cjm_plan(cjm_plan_t *out, int stencil, int nx, int ny, double h,
                    int bc, double tol, const cjm_options *opt);

/* Generic 5-point masks (the code is "totally
 * generic regarding discretization and coordinates", the Laplacian being a
 * per-node mask of coefficients f_W, f_E, f_S, f_N, f_C, tab:ste1; tab:ste2
 * lists the Cartesian, polar and bipolar ones).
 *
 * cjm_plan_mask: a single-GPU plan of nx x ny interior nodes whose operator
 * is set afterwards by cjm_mask_set.  There is no closed form for the
 * spectral bounds of D^-1 A off the Cartesian grid, so the caller passes them
 * (0 < kappa_min < kappa_max; e.g. from cjm_mask_bounds or a dense
 * eigensolver); M, P, the ordering and the weights then follow exactly as in
 * cjm_schedule.  u keeps r = 1 ghost ring (the Dirichlet data), rhs is b in
 * PDE units (A u = b with A the mask), residual norms are of b - A u.  One
 * sweep per launch (options temporal_k / variant / tile_w / stages /
 * resident / band_split are ignored; ctas_per_sm defaults to 8).
 * Errors: INVALID_ARG (sizes, bounds, tol, options), UNSUPPORTED
 * (world_size > 1), OOM, CUDA.  cjm_plan with CJM_STENCIL_MASK is
 * INVALID_ARG. */
cjm_status cjm_plan_mask(cjm_plan_t *out, int nx, int ny, double kappa_min,
                         double kappa_max, double tol, const cjm_options *opt);

/* Upload the mask of a cjm_plan_mask plan: five DEVICE arrays c_W, c_E, c_S,
 * c_N, c_C (PDE units, ny x nx, row-major, pitch ld_c >= nx; node (i,j) at
 * c[(j-1) ld_c + (i-1)]; W/E = first coordinate -/+, S/N = second -/+).  The
 * plan stores a_q = -c_q / c_C (q = W, E, S, N; IEEE division) and c_C
 * (DESIGN R10); the arrays are read during the call only (it synchronises
 * cuda_stream) and stay owned by the caller.  c_C must be non-zero (a zero
 * produces inf / NaN, reported as DIVERGED by the solve).  Must precede
 * cjm_solve / cjm_sweeps / cjm_residual on the plan (else INVALID_ARG); may
 * be called again to change the operator (kappa bounds stay those of the
 * plan).  Errors: INVALID_ARG (not a mask plan, NULL array, ld_c < nx), CUDA. */
cjm_status cjm_mask_set(cjm_plan_t p, const double *cW, const double *cE,
                        const double *cS, const double *cN, const double *cC,
                        long long ld_c, void *cuda_stream);

/* Generic square masks (tab:ste1): "each of its
 * (at most) 24 neighbors spanned by the discretization of the Laplacian can
 * have different numerical factors ... [which] may change as a function of
 * the position of the central node".  radius m = 1: (2m+1)^2 = 9-point masks
 * (the upper, up-to-9-points data structure of tab:ste1); m = 2: 25-point
 * masks (the most generic case, lower part of tab:ste1) -- e.g. the 9- and
 * 17-point Laplacians of Eq. 9-points / Eq. 17-points with per-node factors.
 *
 * cjm_plan_mask_n: as cjm_plan_mask, with u holding m ghost rings
 * ((ny+2m) x (nx+2m), ld_u >= nx + 2m; the outer ring is data too).
 * Errors: INVALID_ARG (radius not 1 or 2, sizes, bounds, tol, options),
 * UNSUPPORTED (world_size > 1), OOM, CUDA. */
cjm_status cjm_plan_mask_n(cjm_plan_t *out, int nx, int ny, int radius, double kappa_min,
                           double kappa_max, double tol, const cjm_options *opt);

/* Upload the mask of a cjm_plan_mask_n plan: planes[q] for q = (dy+m)(2m+1)
 * + (dx+m), dx, dy in -m..m, is a DEVICE array (ny x nx, pitch ld_c >= nx,
 * PDE units) of the coefficient of neighbour (i+dx, j+dy) of node (i,j), or
 * NULL when that neighbour is absent everywhere (it is then neither stored nor
 * read nor added); planes[m(2m+1)+m] = c_C is required.  The plan stores
 * a_q = -c_q / c_C and c_C.  One sweep (DESIGN R11):
 *   J = fma(a_0, u_0, fma(a_1, u_1, ... fma(a_{Q-1}, u_{Q-1}, b/c_C)))
 * over the present q (innermost = largest q), d = J - u_C,
 * u' = fma(w, d, u_C); residual r = c_C d.  The planes array and the arrays
 * it points to are read during the call only (it synchronises cuda_stream).
 * Errors: INVALID_ARG (not a cjm_plan_mask_n plan, NULL planes or centre
 * plane, ld_c < nx), CUDA. */
cjm_status cjm_mask_set_n(cjm_plan_t p, const double *const *planes, long long ld_c,
                          void *cuda_stream);

/* Host-only estimate of the spectral bounds of D^-1 A for a (2m+1)^2 mask
 * (SURVEY A14's numeric fallback; HOST planes laid out as in cjm_mask_set_n,
 * NULL = absent).  No symmetry to exploit: kappa_max by `iters` power-
 * iteration steps on D^-1 A (0 = 2000), kappa_min by as many on
 * kappa_max I - D^-1 A, both from sin(pi i/(nx+1)) sin(pi j/(ny+1)).  An
 * estimate for a symmetrisable D^-1 A: both ends are approached from inside
 * the spectrum, and the kappa_min estimate needs iterations ~ kappa_max /
 * (gap at the bottom of the spectrum) -- fine on coarse grids, not on 4096^2
 * (pass closed-form or safety-widened bounds there).  Cost 2 x iters x nx x
 * ny x (2m+1)^2 on one host core.  Errors: INVALID_ARG (radius, sizes, NULL
 * centre plane, a zero or non-finite c_C, an estimate kappa_min <= 0). */
cjm_status cjm_mask_bounds_n(int nx, int ny, int radius, const double *const *planes,
                             long long ld_c, int iters, double *kappa_min, double *kappa_max);

/* Host-only estimate of the spectral bounds of D^-1 A for a 5-point mask
 * (the numeric fallback; HOST arrays laid out as in
 * cjm_mask_set).  The 5-point grid graph is bipartite, so the spectrum of
 * D^-1 A = I - N is symmetric about 1: kappa_min = 1 - rho(N), kappa_max =
 * 1 + rho(N), rho(N) by `iters` power-iteration steps (0 = 2000) from the
 * positive smooth vector sin(pi i/(nx+1)) sin(pi j/(ny+1)).  An estimate:
 * rho converges from below, so kappa_min may be slightly too large.  Cost
 * iters x nx x ny on one host core.  Errors: INVALID_ARG (sizes, NULL, a zero
 * or non-finite c_C, rho(N) >= 1: D^-1 A not positive definite). */
cjm_status cjm_mask_bounds(int nx, int ny, const double *cW, const double *cE,
                           const double *cS, const double *cN, const double *cC,
                           long long ld_c, int iters, double *kappa_min,
                           double *kappa_max);

/* Static facts of a plan.  Any output pointer may be NULL.
 *   info: kappa_min/max, m_min, cycle_len (other fields zero) and plan_s.
 *   reach: r.  y0 / ny_local: this rank's slab of interior rows (0-based).
 *   host_weights: the P weights in application order (owned by the plan). */
cjm_status cjm_plan_info(cjm_plan_t p, cjm_report *info, int *reach,
                         int *y0, int *ny_local, const double **host_weights);

/* Solve on the device (P:298-309 with the data already resident).
 *   rhs (device, ny_local x nx, pitch ld_rhs), u (device, (ny_local+2r) x
 *   (nx+2r), pitch ld_u): see the conventions above.  All work is enqueued
 *   on `cuda_stream` (a cudaStream_t; NULL = legacy default stream) and the
 *   call synchronises that stream once per cycle to read the residual
 *   (SURVEY section 3).  On return the interior of u holds the iterate after
 *   rep->iterations sweeps: for CJM_OK the first cycle-boundary iterate with
 *   ||r||_2 <= tol ||r_0||_2 (DESIGN R4); for NOT_CONVERGED / STAGNATED /
 *   DIVERGED the last cycle-boundary iterate.  rep (nullable) is filled in
 *   every case.  Multi-GPU: collective, every rank calls it. */
cjm_status cjm_solve(cjm_plan_t p, const double *rhs, long long ld_rhs,
                     double *u, long long ld_u, void *cuda_stream,
                     cjm_report *rep);

/* The solve with the paper's "real error" stop ("we can use the
 * real error instead of a tolerance as the stopping criterion"): stop at the
 * first cycle boundary whose iterate has max |u - u_ref| <= real_tol over the
 * interior.  u_ref (device, ny_local x nx, pitch ld_ref, read only) holds the
 * analytic solution at the nodes.  The plan's tol still sets the cycle
 * length; the residual is still reduced every cycle (report, divergence and
 * stagnation: a real_tol below the discretisation error ends STAGNATED or
 * NOT_CONVERGED).  rep->real_error receives the error of the returned iterate.
 * Errors: INVALID_ARG for a NULL u_ref, ld_ref < nx or real_tol <= 0. */
cjm_status cjm_solve_ref(cjm_plan_t p, const double *rhs, long long ld_rhs,
                         double *u, long long ld_u, const double *u_ref, long long ld_ref,
                         double real_tol, void *cuda_stream, cjm_report *rep);

/* The same solve with HOST buffers: one host->device copy of u and rhs at
 * the start and one device->host copy of the solution at the end (the
 * paper's flow), all inside the call.  Layouts as cjm_solve. */
cjm_status cjm_solve_host(cjm_plan_t p, const double *rhs_host, long long ld_rhs,
                          double *u_host, long long ld_u, void *cuda_stream,
                          cjm_report *rep);

/* Apply `count` scheduled sweeps with no stop test: sweep k (0 <= k < count)
 * uses the weight at cycle position (first + k) mod P.  u (device) is read
 * and overwritten with the result (interior only).  Used to compare a fixed
 * segment of the iteration with the oracle at any size.  rep (nullable)
 * receives sweep_s / sweeps_timed / kernel_launches.  external_halo plans
 * (the caller moves the halos between calls): count <= temporal_k, else
 * INVALID_ARG (a second launch would read stale neighbour rows). */
cjm_status cjm_sweeps(cjm_plan_t p, const double *rhs, long long ld_rhs,
                      double *u, long long ld_u, long long first, long long count,
                      void *cuda_stream, cjm_report *rep);

/* Residual norms of u: ||b - Delta_h u||_2 and ||.||_inf over the (global)
 * interior, in PDE units (fused reduction kernel, allreduced across ranks).
 * Synchronises cuda_stream.  l2 / linf nullable. */
cjm_status cjm_residual(cjm_plan_t p, const double *rhs, long long ld_rhs,
                        const double *u, long long ld_u, void *cuda_stream,
                        double *l2, double *linf);

/* Create an NCCL unique id (128 bytes) for a multi-GPU plan (rank 0). */
cjm_status cjm_get_nccl_id(void *out128);

/* Slab geometry of the 1-D row decomposition (host only): rank g of
 * world_size owns interior rows [floor(g ny / W), floor((g+1) ny / W)). */
cjm_status cjm_slab(int ny, int world_size, int rank, int *y0, int *ny_local);

/* One halo message of the row-slab decomposition (SURVEY section 8(e), row
 * a9).  Rows are numbered in the local iterate buffer of the rank:
 * 0 .. ny_local + 2r - 1, ghost rows included (interior row i at r + i).
 * The rank sends rows [send_row, send_row + rows) to `peer` and receives the
 * peer's message into rows [recv_row, recv_row + rows). */
typedef struct {
    int peer;
    int send_row;
    int recv_row;
    int rows;
} cjm_halo_msg;

/* Host-only halo plan of rank `rank` of `world_size` for a global grid of
 * ny interior rows and halo depth r (the stencil reach, or K r for K-fused
 * launches; 1..16): one message per neighbour slab
 * (0, 1 or 2).  My first r interior rows go to the neighbour above (rank-1),
 * into its last ghost rows; my last r interior rows go to the neighbour below
 * (rank+1), into its first ghost rows.  msgs must hold 2 entries.
 * Errors: INVALID_ARG (sizes, a slab thinner than 2r+1 rows when
 * world_size > 1, r outside 1..16). */
cjm_status cjm_halo_plan(int ny, int r, int world_size, int rank, cjm_halo_msg *msgs,
                         int *nmsgs);

/* Internal buffer layout (host only): the plan's iterate / g buffers have rows
 * of pitch *ld doubles (ld = roundup(nx + 16, 32): 256-byte aligned rows) and
 * interior column i at *col0 + i (col0 = 8; the r ghost columns sit just left
 * and right of the interior).  Row j of the slab (0-based, ghost rows
 * included) starts at element j * ld.  Errors: INVALID_ARG for nx < 1. */
cjm_status cjm_buffer_layout(int nx, long long *ld, int *col0);

/* One halo transfer in elements of the internal buffer layout: send `count`
 * doubles starting at element send_off of my buffer to `peer`, receive the
 * peer's `count` doubles into element recv_off. */
typedef struct {
    int peer;
    long long send_off;
    long long recv_off;
    long long count;
} cjm_halo_xfer;

/* Host-only: the transfers the library's NCCL halo exchange (row a9) issues,
 * verbatim, for rank `rank` of `world_size` on a global grid of nx x ny
 * interior nodes with `depth` halo rows (r, or K r for K-fused launches):
 * cjm_halo_plan's messages as whole rows (ghost columns included) of the
 * internal layout (cjm_buffer_layout; *ld_out nullable).  One ncclSend and
 * one ncclRecv per transfer inside one NCCL group, on the iterate buffer the
 * launch wrote (and once per solve on g when depth > r).  xfers must hold 2
 * entries.  Errors as cjm_halo_plan. */
cjm_status cjm_halo_xfers(int nx, int ny, int depth, int world_size, int rank,
                          cjm_halo_xfer *xfers, int *nxfers, long long *ld_out);

/* Release every device buffer and graph of the plan.  NULL is ok.  The
 * field-sized buffers go to the library's device-buffer cache (reused by the
 * next plan of the same size) and the NCCL communicator back to the
 * communicator cache; cjm_pool_trim frees both. */
cjm_status cjm_plan_destroy(cjm_plan_t p);

/* Return every cached device buffer to the driver (cudaFree) and destroy
 * every idle cached NCCL communicator.  Call when no plan is being created
 * concurrently (multi-GPU: on every rank, at the same point).  cached_bytes_before (nullable)
 * receives the bytes that were cached. */
cjm_status cjm_pool_trim(long long *cached_bytes_before);

const char *cjm_status_str(int status);
const char *cjm_last_error(void);
int cjm_version(void);   /* 100 * major + minor */

#ifdef __cplusplus
}
#endif
#endif /* CJM_H */
