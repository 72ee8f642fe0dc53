/*
 * pins.h -- C ABI of libpins_b200.so: the PINS hot path (arXiv 2502.03749,
 * "PINS: Proximal Iterations with Sparse Newton and Sinkhorn for Optimal
 * Transport") on one B200 (sm_100a).
 *
 * Conventions (all entry points):
 *  - Every array argument is a DEVICE pointer to fp64 (or int32 / int64 where
 *    stated) memory owned by the caller, unless the name ends in _host.  The
 *    library never frees caller memory.  Scratch memory is owned by a
 *    pins_workspace (stream-ordered allocations on the stream passed in).
 *  - `stream` is a cudaStream_t passed as void*; NULL means the legacy default
 *    stream.  Calls are asynchronous w.r.t. the host unless they return host
 *    scalars (documented per call), which synchronise `stream`.
 *  - Return value: PINS_OK (0) or a PINS_ERR_* code; nothing is thrown.  On a
 *    CUDA error the sticky error text is available from pins_last_error().
 *
 * Problem (Eq. (1), lines 41-46):  min <C,X>  s.t.  X e_n = a,
 * X^T e_m = b, X >= 0, with C given either densely or by point coordinates:
 *    C_ij = cost_scale * D_ij,
 *    D_ij = C[i*ldc + j]                       (PINS_COST_DENSE)
 *         = sum_k (x[i*d+k] - y[j*d+k])^2     (PINS_COST_SQEUCLID)
 *         = sum_k |x[i*d+k] - y[j*d+k]|       (PINS_COST_L1)
 * Point kinds recompute D on the fly inside every dense pass (no m x n array).
 *
 * Proximal centre (Eq. (5)-(7), Alg. 2 lines 3 and 16) in factored
 * log form:  C^k = s C - phi (+) psi, i.e.
 *    log X^k_ij = (phi_i + psi_j - s C_ij)/eta        (X^0 = a b^T: s=1,
 *    phi = eta log a, psi = eta log b).
 * Subproblem potentials (f, g) are the paper's; the plan of Eq. (7) is
 *    X~_ij = exp((f_i + phi_i + g_j + psi_j - s C_ij)/eta - 1).
 */
#ifndef PINS_B200_H
#define PINS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PINS_OK 0
#define PINS_ERR_ARG 1        /* invalid argument (sizes, NULL pointers, kinds) */
#define PINS_ERR_CUDA 2       /* CUDA runtime error (see pins_last_error)        */
#define PINS_ERR_NOMEM 3      /* device allocation failed                        */
#define PINS_ERR_NUMERIC 4    /* non-finite value where a finite one is required */

#define PINS_COST_DENSE 0
#define PINS_COST_SQEUCLID 1
#define PINS_COST_L1 2

typedef struct pins_problem {
    int64_t m, n;            /* sizes, m >= 1, n >= 1                              */
    int32_t cost_kind;       /* PINS_COST_*                                        */
    int32_t d;               /* point dimension (1..16) for point kinds            */
    const double *C;         /* DENSE: device m x n, row-major, leading dim ldc    */
    int64_t ldc;             /* >= n                                               */
    const double *x;         /* points: device m x d row-major (integer-valued for */
    const double *y;         /*   exact costs; any finite values are accepted)     */
    double cost_scale;       /* C_ij = cost_scale * D_ij  (> 0)                    */
    const double *a;         /* device m, > 0, sum 1                               */
    const double *b;         /* device n, > 0, sum 1                               */
    double eta;              /* entropic / proximal parameter, > 0                 */
} pins_problem;

/* Solver parameters; semantics identical to oracle/pins_oracle.py Params.
 * Defaults (pins_default_params) follow PAPER.md Appendix A.2 (lines 477-485). */
typedef struct pins_params {
    int32_t K;               /* max EPPA (outer) iterations               (500)   */
    int32_t outer_rule;      /* 0 rel. change, 1 halving, 2 geometric tail,
                                3 certified: LP gap <= outer_tol |obj| (0)   */
    double outer_tol;        /* outer tolerance                           (1e-4)  */
    int32_t T1;              /* max Sinkhorn sweeps per subproblem        (50000) */
    double sink_tol;         /* Sinkhorn phase: ||grad P||_1 threshold    (6.3e-4)*/
    int32_t T2;              /* max Newton iterations per subproblem      (20)    */
    double newton_tol;       /* Newton phase: ||grad P||_1 threshold      (1e-8)  */
    double theta;            /* sparsify: keep X~_ij >= theta/(m n)       (1e-4)  */
    double cg_tol;           /* CG relative-residual floor                (1e-6)  */
    double cg_forcing;       /* rtol = clamp(cg_forcing*newton_tol/||g||_1, cg_tol, 0.5) (0.5) */
    int32_t cg_maxit;        /* (1000) */
    double mu_rel;           /* damping mu = mu_rel * max diagonal        (1e-10) */
    double armijo_c;         /* (1e-4) */
    double beta;             /* backtracking factor (0.5) */
    int32_t max_backtracks;  /* (30) */
    int32_t warm_start;      /* 0 zero, 1 carry (f,g) across outer iterations, 2 linear
                                extrapolation 2x^k - x^{k-1} kept only if it needs no
                                Sinkhorn phase (R7)               (1)    */
} pins_params;

void pins_default_params(pins_params *p);

/* Opaque scratch owner (row buffers, CSR/CSC, column partials, CG vectors).
 * Every entry point that takes a pins_problem rebuilds the workspace's
 * derived problem data (padded point copies, exactness decision, chunk-skip
 * certificates) at entry, so one workspace may serve many problems.       */
typedef struct pins_workspace pins_workspace;
int pins_workspace_create(pins_workspace **ws);
void pins_workspace_destroy(pins_workspace *ws);

/* Last error message for this thread (static storage, never NULL). */
const char *pins_last_error(void);

/* Initialise the proximal centre to X^0 = a b^T: s=1, phi = eta log a,
 * psi = eta log b.  phi (m), psi (n) device, caller-owned.                   */
int pins_center_init(const pins_problem *pb, double *phi, double *psi, double *s_host,
                     void *stream);

/* Proximal-centre update, Alg. 2 line 16 then line 3:
 * X^{k+1} = X~(f, g) in log form:  phi += f,  psi += g - eta,  s += 1.       */
int pins_center_update(const pins_problem *pb, double *phi, double *psi, double *s_host,
                       const double *f, const double *g, void *stream);

/* One log-domain Sinkhorn sweep in place, Alg. 2 lines 5-6:
 *   f <- eta(log a + 1) - eta LSE_j((g_j - C^k_ij)/eta)
 *   g <- eta(log b + 1) - eta LSE_i((f_i - C^k_ij)/eta)   (with the new f).
 * Two launches of the half-sweep kernel (row orientation, then column
 * orientation with the new f); each merges its column splits in its own
 * last-arriving CTA (no host round trip).  Asynchronous.                     */
int pins_sinkhorn_sweep(pins_workspace *ws, const pins_problem *pb, const double *phi,
                        const double *psi, double s, double *f, double *g, void *stream);

/* The Sinkhorn phase of Alg. 2 (lines 4-8): sweeps of
 * pins_sinkhorn_sweep until ||grad P^k||_1 <= tol or max_sweeps sweeps; stops
 * at exactly the first iterate whose residual is <= tol (the test runs on
 * the device; batches of sweeps are queued without host round trips).
 * A phase longer than 7 sweeps continues with absorbed kernel-matrix sweeps
 * (DESIGN.md section 5): inside one phase only the column potentials move, so
 * exp(x_ij - r_i) = K_ij u_j with K fixed since the last record pass; a
 * half-sweep is then one exponential per column and one FMA per listed entry
 * of a sliced-ELL copy of K (entries within the log-sum-exp cut of the row
 * maximum, plus a margin; a per-(row, split) certificate proves that unlisted
 * entries stay below the cut, failed units are scanned densely).  Same sums as
 * the log-domain sweep up to rounding (tested against the oracle and against
 * the dense sweeps); environment PINS_KSWEEP=0 keeps every sweep dense.
 * *sweeps_host = sweeps done, *res_host = final ||grad P^k||_1.  Synchronises. */
int pins_sinkhorn(pins_workspace *ws, const pins_problem *pb, const double *phi, const double *psi,
                  double s, double *f, double *g, double tol, int32_t max_sweeps, int32_t *sweeps_host,
                  double *res_host, void *stream);

/* Evaluation pass at (f, g): plan X~ of Eq. (7), its row sums r (m) and column
 * sums c (n) (either may be NULL), the gradient norm and objectives.  Host
 * scalars (synchronises); out_host must hold at least 6 doubles:
 * out_host[0] = ||a - r||_1 + ||b - c||_1 (= ||grad P^k||_1, Eq. (9)),
 * [1] = sum X~,  [2] = <C, X~>,  [3] = P^k(f,g) (Eq. (8)),  [4] = nnz of the
 * sparsified block (0 if tau == 0),  [5] = max_ij z_ij, z = log X~ (over the
 * entries the pass evaluates).  If tau > 0 the plan block is also sparsified
 * (X~_ij >= tau) into the workspace CSR (and CSC).                           */
int pins_evaluate(pins_workspace *ws, const pins_problem *pb, const double *phi,
                  const double *psi, double s, const double *f, const double *g,
                  double tau, double *r, double *c, double *out_host, void *stream);

/* The CSR produced by the last pins_evaluate(tau > 0) / pins_newton_step
 * (Alg. 2 line 11, reading R3): row-major, columns
 * ascending, entries X~_ij >= tau.  *nnz_host, *m_host receive the sizes;
 * if rowptr (m+1, int64), colidx (int32) and val (fp64) are non-NULL the CSR
 * is copied into them (cap >= nnz required, else PINS_ERR_ARG).  Synchronises. */
int pins_get_csr(pins_workspace *ws, int64_t *rowptr, int32_t *colidx, double *val, int64_t cap,
                 int64_t *nnz_host, int64_t *m_host);

/* Sparsify a caller-given dense plan block P (device m x n, leading dim ldp):
 * CSR of P_ij >= tau (reading R3), columns ascending, values
 * copied bitwise.  Warp-ballot compaction (sparsify_*_kernel), separate from
 * the evaluation pass's fused compaction (which sparsifies X~(f, g) without
 * materialising it; see pins_evaluate).  *nnz_host always receives nnz; if
 * rowptr (m+1, int64), colidx (int32), val (fp64) are non-NULL they receive
 * the CSR (cap >= nnz required, else PINS_ERR_ARG).  Invalidates the
 * workspace CSR of the last evaluation.  Synchronises.                      */
int pins_sparsify_dense(pins_workspace *ws, int64_t m, int64_t n, const double *P, int64_t ldp,
                        double tau, int64_t *rowptr, int32_t *colidx, double *val, int64_t cap,
                        int64_t *nnz_host, void *stream);

/* Jacobi-preconditioned CG (reading R5) on
 *   M = [[diag(dr) , Xs ], [Xs^T, diag(dc)]] + mu I,   M x = rhs
 * with Xs given as CSR (rowptr int64 m+1, colidx int32, val fp64, nnz).
 * rhs, x: device (m+n); x is overwritten (start 0).  One cooperative
 * persistent launch; iterations and final relative residual returned on the
 * host (synchronises).                                                        */
int pins_cg(pins_workspace *ws, int64_t m, int64_t n, const int64_t *rowptr,
            const int32_t *colidx, const double *val, int64_t nnz, const double *dr,
            const double *dc, double mu, const double *rhs, double *x, double rtol,
            int32_t maxit, int32_t *iters_host, double *relres_host, void *stream);

/* One sparse Newton iteration on subproblem k, Alg. 2 lines 10-14
 * (PAPER.md:173-180): evaluate + sparsify (tau = theta/(mn)), CG on the
 * sparsified Hessian, backtracking line search, update (f, g) in place.
 * info_host: [0] grad l1 before, [1] grad l1 after, [2] alpha, [3] CG iters,
 * [4] CG rel. residual, [5] nnz, [6] line-search trials.  Synchronises.       */
int pins_newton_step(pins_workspace *ws, const pins_problem *pb, const pins_params *prm,
                     const double *phi, const double *psi, double s, double *f, double *g,
                     double *info_host, void *stream);

/* LP residuals of the plan X~(f,g) at centre (phi,psi,s) (reading R8):
 * res_host[0] = ||Xe-a||_1 + ||X^Te-b||_1, [1] = max(0, max_ij u_i+v_j-C_ij)
 * with u = (f+phi)/s, v = (g+psi-eta)/s, [2] = <C,X>, [3] = <a,u>+<b,v>,
 * [4] = [2]-[3].  u, v (device m, n) written if non-NULL.  Synchronises.     */
int pins_residuals(pins_workspace *ws, const pins_problem *pb, const double *phi,
                   const double *psi, double s, const double *f, const double *g,
                   double *u, double *v, double *res_host, void *stream);

/* LP certificate of the plan X~(f,g) at centre (phi, psi, s) (reading R11,
 * DESIGN.md §3; LP duality of Eq. (1)): evaluation with the
 * plan block sparsified at tau = 1e-12/(m n) (prm is not used for it); the
 * maximum-weight spanning forest of that support (the LP optimum is a vertex, whose
 * support is a forest); tree duals u_i + v_j = C_ij on the forest; row then
 * column c-transforms u_i = min_j C_ij - v_j, v_j = min_i C_ij - u_i (dual
 * feasible by construction); the entropic duals are the fallback candidate.
 * u (m), v (n): device outputs, may be NULL.  cert_host (>= 8 doubles):
 * [0] ||Xe-a||_1 + ||X^Te-b||_1, [1] <C,X>, [2] <a,u> + <b,v> (<= LP*),
 * [3] gap = [1] - [2], [4] measured max(0, max_ij u_i + v_j - C_ij),
 * [5] forest edges (0: no forest built, m + n > 26000), [6] 1 if the forest's
 * duals gave the bound, [7] nnz of the sparsified support.  Synchronises.  */
int pins_lp_certificate(pins_workspace *ws, const pins_problem *pb, const pins_params *prm,
                        const double *phi, const double *psi, double s, const double *f, const double *g,
                        double *u, double *v, double *cert_host, void *stream);

/* Materialise X~(f,g) densely (device m x n, leading dim ldx).  Asynchronous. */
int pins_plan(const pins_problem *pb, const double *phi, const double *psi, double s,
              const double *f, const double *g, double *X, int64_t ldx, void *stream);

/* Output of pins_solve.  Device arrays are caller-owned (f, g, phi, psi: sizes
 * m, n, m, n; u, v optional).  Scalars are written on the host.
 * LP KKT of the returned plan X = X~(f, g) (reading R11):
 * kkt = primal residual, dual_inf = measured dual infeasibility of (u, v),
 * gap = <C, X> - lp_dual_obj; (u, v) are CERTIFIED duals -- dual feasible by
 * construction (c-transforms of the tree duals of the plan's maximum-weight
 * spanning forest, or of the entropic duals, whichever bound is larger), so
 * lp_dual_obj <= LP* (weak duality) and gap bounds the objective error.     */
typedef struct pins_result {
    double *f, *g;           /* last subproblem potentials (device)              */
    double *phi, *psi;       /* proximal centre log form (device)                */
    double *u, *v;           /* certified LP duals (device, may be NULL)         */
    double s;                /* centre scale s_K                                 */
    double obj;              /* <C, X>  (primal objective of the returned plan)  */
    double dual_obj;         /* P^k(f,g) of the last subproblem (Eq. (8))        */
    double lp_dual_obj;      /* <a,u> + <b,v>  (a certified lower bound on LP*)  */
    double kkt;              /* ||Xe-a||_1 + ||X^Te-b||_1  (primal residual)     */
    double dual_inf;         /* max(0, max_ij u_i + v_j - C_ij)  (measured)      */
    double gap;              /* obj - lp_dual_obj                                */
    int32_t outer_iters, sweeps, newton_iters, cg_iters, status; /* status 0 = converged, 1 = budget */
    int32_t certificates;    /* LP certificates built during the solve           */
    int32_t cert_tree;       /* 1: the returned duals are the tree-basis ones    */
    double *obj_trace_host;  /* optional host array of length >= K (may be NULL) */
    double seconds;          /* host wall time of the solve                      */
} pins_result;

/* Full PINS solve, Algorithm 2.  Synchronises.
 * Point costs are solved on a copy permuted into Morton order of the
 * coordinates (locality for the dense passes) and the potentials are scattered
 * back, so every output is in the caller's order.  The Newton systems use the
 * spanning-tree preconditioned CG when m + n <= 26000 and nnz <= 4e5 (falling
 * back to the Jacobi-Schur cluster CG after a slow tree solve), else Jacobi CG
 * on the whole GPU; the cluster tree-PCG starts from the
 * A-norm-optimal multiple of the previous Newton direction.  Dense passes over
 * integer point clouds skip 32-column chunks that a drift certificate proves
 * empty (bit-identical results).  Development knobs
 * (environment): PINS_CG = tree | treecl | cluster | grid forces a solver,
 * PINS_NO_TC=1 turns the tensor-core cross term off, PINS_NO_REORDER=1 the
 * Morton permutation, PINS_NO_TILESKIP=1 chunk skipping, PINS_NO_X0=1 the PCG
 * warm start; PINS_TREE_NNZ_MAX=<n> moves the tree-PCG nnz cap;
 * PINS_TRACE=<file> writes one line per outer iteration, PINS_SKIP_STATS=1
 * prints chunk-skip totals to stderr.                                        */
int pins_solve(const pins_problem *pb, const pins_params *prm, pins_result *res, void *stream);

/* pins_solve on a caller-owned workspace (reused across solves: no per-solve
 * workspace creation, pinned-buffer allocation or scratch growth).  The
 * workspace's derived problem data are rebuilt at entry.  Synchronises.     */
int pins_solve_ws(pins_workspace *ws, const pins_problem *pb, const pins_params *prm, pins_result *res,
                  void *stream);

/* End-to-end solve from HOST memory (bench.py's e2e leg): pb_host is a
 * pins_problem whose C / x / y / a / b point to HOST memory (pinned for the
 * asynchronous path; pageable works but synchronises).  The instance is
 * copied host->device on `stream` into library-owned stream-ordered device
 * memory, pins_solve runs, and the outputs requested in res_host (f, g, phi,
 * psi, u, v: HOST pointers, each may be NULL) are copied device->host.
 * io_bytes_host[0] / [1] receive the host->device / device->host byte counts.
 * Device memory is released before return.  Synchronises.                    */
int pins_solve_host(const pins_problem *pb_host, const pins_params *prm, pins_result *res_host,
                    int64_t *io_bytes_host, void *stream);

/* ------------------------------------------------------------------ profiling
 * Device-time profile of this library's own kernel launches (used by bench.py
 * for the roofline of the dominant kernel).  Every launch is counted per
 * class; while enabled, each launch is bracketed by a pair of CUDA events on
 * the stream it is launched on (adds ~2 event records per launch).
 * pins_prof_read synchronises on the pending events and returns, for a class,
 * the number of launches and the summed device milliseconds since the last
 * pins_prof_reset.  Process-global, not thread-safe.                          */
#define PINS_PROF_SWEEP_ROW 0   /* Sinkhorn row pass (f update)                */
#define PINS_PROF_SWEEP_COL 1   /* Sinkhorn column pass (g update)             */
#define PINS_PROF_EVAL 2        /* plan evaluation / sparsify / trial pass     */
#define PINS_PROF_REDUCE 3      /* column-partial and scalar reductions        */
#define PINS_PROF_CSR 4         /* CSR / CSC construction                      */
#define PINS_PROF_CG 5          /* conjugate gradient                          */
#define PINS_PROF_VEC 6         /* small vector kernels                        */
#define PINS_PROF_PLAN 7        /* dense plan materialisation                  */
#define PINS_PROF_KSWEEP 8      /* absorbed kernel-matrix half-sweep (ELL walk)   */
#define PINS_PROF_SWEEP_AUX 9   /* list modes: record passes (incl. their no-op launches), sort, ELL build, fallback, merge */
#define PINS_PROF_NCLASS 10
void pins_prof_enable(int32_t on);
void pins_prof_reset(void);
int pins_prof_read(int32_t cls, int64_t *launches, double *ms);
/* Work attributed to a class since the last reset: for PINS_PROF_CG the bytes
 * of every iteration's sparse products and vector streams (24 B x nnz + 80 B x
 * (m + n) per iteration, counted by the host); for PINS_PROF_SWEEP_ROW (all
 * half-sweeps) and PINS_PROF_EVAL (sum passes) the number of plan entries that
 * survived the skip test and were evaluated exactly (counted on the device
 * while profiling is enabled; synchronises); for PINS_PROF_KSWEEP the listed
 * entries the ELL walks read (12 B each: int32 column + fp64 kernel value);
 * 0 for other classes.                                                      */
int pins_prof_read_work(int32_t cls, double *work);

#ifdef __cplusplus
}
#endif
#endif /* PINS_B200_H */
