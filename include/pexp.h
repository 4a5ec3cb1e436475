/*
 * pexp.h — C ABI of the B200-native Paraexp-EBK hot path (arXiv 1509.04567).
 *
 * What it computes (PAPER.md = "P:<line>", readings #k = DESIGN.md §3):
 *   Linear:  u' = A u + g(t), u(0) = u0, A = nu*D2 - a*D1,
 *            solved by Paraexp superposition (Fig. 2) with one
 *            exponential-block-Krylov (EBK) evaluation per subinterval:
 *            truncated SVD of the sampled shifted source, shift-and-invert block
 *            Arnoldi, projected exponential, superposition of nonhomogeneous and
 *            homogeneous parts.
 *   Burgers: u' = nu*D2 u - u∘(D1 u) (f = 0), solved by waveform relaxation
 *            with per-subinterval averaged Jacobians (§2.4, Fig. 5 P:428-444;
 *            Eq.(sourceParallel) read as in reading #2).
 *
 * Conventions for every call:
 *   - All array arguments are CALLER-OWNED, fp64, contiguous, last index fastest.
 *     Pointers documented "dev" are CUDA device pointers; "host" are host pointers.
 *     The library never frees caller memory.
 *   - All device work is enqueued on the stream given in pexp_options.stream
 *     (a cudaStream_t; NULL = legacy default stream).  A pexp_solve_* call returns
 *     after its work has completed.  It synchronises that stream at the end and at
 *     the host-side control points listed in DESIGN.md §5.7 (block-width selection,
 *     Krylov convergence checks, WR stop test); pexp_stats.host_syncs counts them.
 *   - Device scratch comes from the caller: query pexp_workspace_bytes(), allocate
 *     (e.g. a torch uint8 CUDA tensor), bind with pexp_set_workspace().  The library
 *     never calls cudaMalloc for scratch.
 *   - Errors: every call returns a pexp_status; nothing throws across the ABI.
 *     On error the output arrays are unspecified and pexp_last_error() returns a
 *     NUL-terminated message owned by the context (valid until the next call on it).
 *   - Grids (reading #15): periodic x_i = i/n, dx = 1/n; Dirichlet x_i = (i+1)/(n+1),
 *     dx = 1/(n+1), zero boundary values.  Sample nodes (reading #9): with dT = T/P,
 *     t_{j,i} = j*dT + i*(dT/(s-1)), j = 0..P-1, i = 0..s-1 (endpoints included); with
 *     pexp_options.node_rule = 1 the Chebyshev-Lobatto points of each subinterval instead.
 *     pexp_sample_times returns the nodes of the context's rule.
 */
#ifndef PEXP_H
#define PEXP_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PEXP_API __attribute__((visibility("default")))
#else
#define PEXP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pexp_ctx pexp_ctx; /* opaque, owned by the library */

typedef enum {
  PEXP_OK = 0,
  PEXP_EINVAL = 1,    /* invalid argument (message says which)                        */
  PEXP_ENOMEM = 2,    /* workspace missing or too small                              */
  PEXP_ECUDA = 3,     /* a CUDA runtime error (message carries cudaGetErrorString)    */
  PEXP_ENOCONV = 4,   /* Krylov column cap k_max reached above tolerance              */
  PEXP_EDIVERGED = 5, /* WR iterate non-finite or its change grew > 1e3x      */
  PEXP_EPIVOT = 6     /* shift-and-invert factorisation: a pivot that is zero relative to
                         its row (|d_i| <= 1e-13 (|T_ii| + |l_i c_{i-1}|)) or non-finite    */
} pexp_status;

typedef enum { PEXP_BC_PERIODIC = 0, PEXP_BC_DIRICHLET = 1 } pexp_bc;

/* Method options.  A zero-initialised struct means "defaults". */
typedef struct {
  int32_t s;              /* source samples per subinterval, >= 4 (default 32)           */
  int32_t node_rule;      /* 0 = uniform nodes incl. endpoints, p(t) = not-a-knot cubic spline (default);
                             1 = Chebyshev-Lobatto nodes t_{j,i} = j*dT + (dT/2)(1 - cos(pi i/(s-1)))
                             (P:451), p(t) = the degree-(s-1) interpolant through them, integrated
                             through its 12-term Taylor polynomials on s-1 uniform pieces (DESIGN.md
                             §3 #23).  Linear solves only; needs k_max + 12 s <= 1024          */
  double svd_tau_factor;  /* truncation tau_svd = factor*tol relative to sigma_1 (0.01)  */
  double stop_factor;     /* Krylov stop eta = factor*tol (default 0.1; DESIGN.md §3 #6)  */
  int32_t restart_blocks; /* restart a Krylov cycle after this many block steps (P:451:
                             "restarted every 20 iterations"); 0 = default 20; < 0 = only
                             when the basis capacity basis_cols is full.  Exact nested
                             restart, DESIGN.md §3 #5                                       */
  int32_t k_max;          /* total Krylov dimension per evaluation over all restart
                             cycles (default 256; k_max + 4 s <= 1024)                     */
  void* stream;           /* cudaStream_t; NULL = legacy default stream                  */
  int32_t stop_rule;      /* 0 = shift-and-invert residual ||(I-gamma A)^{-1} r(t)|| (default),
                             1 = true residual ||r(t)|| = ||A y + U p - y'|| (DESIGN.md §3 #6) */
  int32_t basis_cols;     /* basis columns kept per evaluation in one cycle (device memory:
                             8 n basis_cols bytes per evaluation); 0 = k_max               */
  int32_t eval_chunk;     /* nonhomogeneous EBK evaluations resident at once (the basis
                             memory is eval_chunk * basis_cols * n * 8 bytes); 0 = all      */
  int32_t route;          /* block Arnoldi route: 0 = auto (fused cluster step when the
                             step's panels fit shared memory, else the streaming route),
                             1 = always the streaming route (full-grid TMA/DMMA kernels per
                             product), 2 = fused step where it fits       */
  double defl_tol;        /* deflation: a new Krylov column is dropped when block Gram-
                             Schmidt leaves < defl_tol of its pre-orthogonalisation norm
                             (default 1e-10; DESIGN.md §3 #22)                            */
  double piv_tol;         /* in-block Cholesky-QR: smallest accepted scaled pivot
                             (default 1e-14)                               */
  int32_t hom_group;      /* linear homogeneous legs sharing one block Krylov space
                             (default 8, at most 16)                       */
  int32_t width_buckets;  /* 0 = default (on): evaluations grouped by retained rank m_j run
                             with their own block width; -1 = off (every evaluation padded
                             to max_j m_j).                                 */
  double scan_gamma_factor; /* Burgers homogeneous scan: its shift-and-invert parameter is
                             scan_gamma_factor * gamma_j (own factorisation when != 1); 0 = default 1.
                             Route only (reading #4)                                        */
  double gamma_factor;    /* shift-and-invert parameter of the nonhomogeneous evaluations:
                             gamma = gamma_factor * dT/10 (Burgers: before the cap of reading #4);
                             0 = default 1.  Route only                                       */
} pexp_options;

/* Per-solve statistics (host memory, caller-owned). */
typedef struct {
  int32_t wr_iters;        /* WR iterations performed (Burgers), 0 for linear          */
  double wr_last_delta;    /* last max-norm change delta_k (Burgers)                  */
  int32_t max_m;           /* largest block width m_j (retained singular values)      */
  int32_t max_k;           /* largest Krylov dimension reached                          */
  int32_t restarts;        /* restart cycles performed                                 */
  double best_residual;    /* worst relative residual at the last check               */
  float ms_total;          /* device time of the call (CUDA events), ms                */
  int32_t evals;           /* nonhomogeneous EBK evaluations performed                 */
  int32_t kernel_launches; /* kernels this library launched during the call            */
  int32_t host_syncs;      /* host<->device synchronisations the call performed         */
  double delta_hist[64];   /* Burgers: delta_k of WR iterations k = 1..min(wr_iters, 64)  */
  /* Optional per-evaluation records (host arrays, caller-owned, NULL = not recorded).
   * Linear: index b*P + j (one EBK evaluation per subinterval j of problem b).
   * Burgers: index k*P + j for WR iteration k < max_wr_iters, subinterval j.
   * m_j: retained source rank (block width); k_j: total Krylov dimension at convergence
   * (all restart cycles); gamma_j: shift-and-invert parameter (reading #4). */
  int32_t* m_j;
  int32_t* k_j;
  double* gamma_j;
  int32_t* kscan_j;        /* Burgers only (nullable): Krylov dimension of the homogeneous scan
                              step of subinterval j (index k*P + j; -1 = waveform written in-scan) */
  float ms_nonhom;         /* device time of the nonhomogeneous parts (source assembly, SVD, EBK of
                              all subintervals at once): the paper's tau_1 with every subinterval
                              concurrent                                            */
  float ms_hom;            /* device time of the homogeneous parts and the superposition (linear:
                              grouped legs; Burgers: the scan + waveform update): tau_2        */
  double scan_steps;       /* Burgers: Arnoldi steps the homogeneous scan performed (all subintervals
                              and iterations), projected-problem checks of its checker CTA, and
                              SM cycles that CTA spent in them (diagnostics)   */
  double scan_checks;
  double scan_check_cycles;
} pexp_stats;

/* Create a context for one spatial operator A = nu*D2 - a*D1 on n points.
 * n >= 3; nu >= 0; bc periodic or Dirichlet.  opt may be NULL (defaults).
 * Host-only: no device work.  *ctx is set to NULL on error. */
PEXP_API pexp_status pexp_create(pexp_ctx** ctx, int64_t n, pexp_bc bc, double nu, double a,
                        const pexp_options* opt);

/* Batched variant (config C4): `batch` independent problems sharing n and bc, each
 * with its own nu_host[b] >= 0 and a_host[b] (host arrays of length batch). */
PEXP_API pexp_status pexp_create_batched(pexp_ctx** ctx, int64_t n, pexp_bc bc, int32_t batch,
                                const double* nu_host, const double* a_host,
                                const pexp_options* opt);

PEXP_API void pexp_destroy(pexp_ctx* ctx);
PEXP_API const char* pexp_last_error(const pexp_ctx* ctx);

/* Sample times t_{j,i} (header comment) written to t_host[j*s + i], length P*s. */
PEXP_API pexp_status pexp_sample_times(const pexp_ctx* ctx, double T, int32_t P, double* t_host);

/* node_rule = 1 only (host-only, no device work): the linear map from the s values of a coefficient row at
 * the Chebyshev-Lobatto nodes of a subinterval of length dT to the Taylor coefficients p^(q)(sigma_i),
 * q = 0..11, of the degree-(s-1) interpolant at the uniform piece starts sigma_i = i dT/(s-1), i = 0..s-2
 * (DESIGN.md §3 #23):  D_host[(i*12 + q)*s + k], (s-1)*12*s doubles.  Returns the number of Taylor terms
 * (12) or 0 for a context with node_rule = 0 / bad arguments. */
PEXP_API int32_t pexp_chebyshev_taylor_matrix(const pexp_ctx* ctx, double dT, double* D_host);

/* Bytes of device scratch needed for solves with P subintervals.
 * kind: 0 = pexp_solve_linear (and the stage entry points), 1 = pexp_solve_burgers,
 * 2 = the larger of both.  Returns 0 for invalid arguments. */
PEXP_API size_t pexp_workspace_bytes(const pexp_ctx* ctx, int32_t P, int32_t kind);
/* Bind caller-owned device scratch (>= pexp_workspace_bytes, 256-byte aligned). */
PEXP_API pexp_status pexp_set_workspace(pexp_ctx* ctx, void* dev_ptr, size_t bytes);

/* Linear Paraexp-EBK solve (Fig. 2).
 *   u0  dev [batch][n]          initial state
 *   src dev [batch][P][s][n]    g(x, t_{j,i}) at the sample nodes (header comment)
 *   T > 0, P >= 1, 1e-14 <= tol <= 1e-2
 *   out dev [batch][P][n]       u(T_1), ..., u(T_P)   (reading #12)
 *   st  host, nullable */
PEXP_API pexp_status pexp_solve_linear(pexp_ctx* ctx, const double* u0, const double* src, double T,
                              int32_t P, double tol, double* out, pexp_stats* st);

/* Burgers waveform relaxation (Fig. 5); requires a periodic context with
 * batch 1; the call's nu is used, the context's nu and a are ignored (reading #18).
 *   u0  dev [n];  out dev [P][n] = u_K(T_1..T_P) after K iterations, K the first k with
 *   delta_k = max|u_{k+1}-u_k| < 1e-6 (reading #13) or K = max_wr_iters. */
PEXP_API pexp_status pexp_solve_burgers(pexp_ctx* ctx, const double* u0, double nu, double T, int32_t P,
                               double tol, int32_t max_wr_iters, double* out, pexp_stats* st);

/* Forced Burgers u' = nu*D2 u - u∘(D1 u) + f(x,t) (Eq.(burgersEq); the paper's
 * sawtooth and multiscale workloads).  As pexp_solve_burgers, plus
 *   f   dev [P][s][n]  forcing samples f(x, t_{j,i}) at the sample nodes (header comment),
 *                      nullable (NULL = unforced).  The sample at T_j appears twice: as
 *                      f[j-1][s-1] and f[j][0].
 * The forcing enters the shifted source of Eq.(sourceParallel) P:312 (reading #2) as
 * g_k(t) = -u_k∘(D1 u_k) + f(t); nothing else changes. */
PEXP_API pexp_status pexp_solve_burgers_forced(pexp_ctx* ctx, const double* u0, const double* f, double nu,
                                      double T, int32_t P, double tol, int32_t max_wr_iters,
                                      double* out, pexp_stats* st);

/* ---- Stage entry points (same kernels as the solves; used by stage-parity tests) ---- */

/* Linear solve with its stage results exposed (stage parity of SURVEY §8(c).5).  As
 * pexp_solve_linear, plus
 *   vstart dev [batch][P][n], nullable: when given, the nonhomogeneous stage is skipped and the
 *          homogeneous legs start from v_j(T_j) := vstart[b][j-1] (src may then be NULL);
 *   vend   dev [batch][P][n], nullable: receives v_j(T_j), j = 1..P, the nonhomogeneous parts at
 *          their subinterval ends (Eq.(linivpSubproblem));
 *   legs   dev [batch][G][P][n], nullable, G = ceil((P-1)/hom_group): legs[b][g][i] receives the
 *          sum over the legs j of group g (j = g*hom_group+1 ...) of exp((T_{i+1}-T_j)A) v_j(T_j)
 *          for T_{i+1} > T_j (Fig. 2 "Solve homogeneous part"); with hom_group = 1 group g
 *          holds the single leg j = g+1. */
PEXP_API pexp_status pexp_solve_linear_stages(pexp_ctx* ctx, const double* u0, const double* src,
                                     const double* vstart, double T, int32_t P, double tol, double* out,
                                     double* vend, double* legs, pexp_stats* st);

/* One waveform-relaxation map u_k -> u_{k+1} = F(u_k) (Eq.(ivpSubproblem)/(updateSolution)
 * P:326-335; one pass of Fig. 5's loop body) from a caller-supplied iterate:
 *   Uk   dev [P][s][n]  u_k at the sample nodes;  Unew dev [P][s][n] receives u_{k+1};
 *   out  dev [P][n]     u_{k+1}(T_1..T_P);  f nullable (pexp_solve_burgers_forced);
 *   st->wr_last_delta = max|u_{k+1} - u_k|. */
PEXP_API pexp_status pexp_wr_map(pexp_ctx* ctx, const double* u0, const double* f, const double* Uk, double nu,
                        double T, int32_t P, double tol, double* Unew, double* out, pexp_stats* st);

/* One batch of shift-and-invert solves (subsystem 1): x = (I - gamma*A_b)^{-1} rhs for
 * problem b of the context, every column c of rhs dev [ncols][n] -> x dev [ncols][n]. */
PEXP_API pexp_status pexp_sai_solve(pexp_ctx* ctx, int32_t b, double gamma, const double* rhs,
                           int32_t ncols, double* x);

/* Truncated SVD stage (subsystem 3) of E sample matrices G dev [E][s][n] (rows = time
 * samples).  Writes m_host[E] (retained rank), sigma dev [E][s] (singular values,
 * descending) and the projection P dev [E][s][n] = U U^T G (rank-m part). */
PEXP_API pexp_status pexp_source_svd(pexp_ctx* ctx, const double* G, int32_t E, double tol,
                            int32_t* m_host, double* sigma, double* proj);

/* Batched Pade-13 scaling-and-squaring exponential (subsystem 4) of E dense N x N
 * matrices A dev [E][N][N] (column-major per matrix) -> X dev [E][N][N]. */
PEXP_API pexp_status pexp_expm_batched(pexp_ctx* ctx, const double* A, int32_t E, int32_t N, double* X);

/* ---- Live per-kernel-class profiler (diagnostics; used by bench.py's roofline) ----
 * Classes: 0 SaI solve, 1 X^T Y projections/Grams (incl. reduce), 2 tall-skinny combine,
 * 3 projected problem (Pade-13 expm + chaining + residual), 4 small dense (eig, Cholesky,
 * one-sided SVD, spline), 5 stencil / assembly / superposition, 6 factorisation,
 * 7 fused Arnoldi step (SaI solve + BCGS2 + in-block QR, one cluster per evaluation),
 * 8 Burgers homogeneous scan (persistent), 9 grouped homogeneous legs' projected problem,
 * 10 streaming-route projection [V W]^T W (TMA + DMMA), 11 streaming-route update W -= V H,
 * 12 Burgers waveform update after the scan (all subintervals in parallel).
 * pexp_profile_enable(1) clears and starts recording CUDA events around every launch
 * (on the launch stream), with the launch's ALGORITHMIC bytes and flops;
 * pexp_profile_read() synchronises the device, fills per-class sums (ms, bytes, flops,
 * launches; arrays of length ncat, host) and clears; returns the number of classes. */
PEXP_API void pexp_profile_enable(int32_t on);
PEXP_API int32_t pexp_profile_read(int32_t ncat, double* ms, double* bytes, double* flops, int32_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* PEXP_H */
