// kernels.cuh — data structures and launch wrappers shared by the pexp sources.
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace pexp {

constexpr int KSMALL_MAX = 1024;  // max Krylov columns (K + m) of one projected problem

// Per-call numerical / routing configuration, set from pexp_options at the start of every
// C-ABI call (thread-local: concurrent calls on different host threads do not interfere).
struct CallCfg {
  double defl = 1e-10;     // pexp_options.defl_tol
  double piv_tol = 1e-14;  // pexp_options.piv_tol
  int route = 0;           // pexp_options.route (0 auto, 1 streaming, 2 fused where it fits)
  int hom_group = 8;       // pexp_options.hom_group
  int buckets = 1;         // pexp_options.width_buckets (0: pad every evaluation to max m_j)
  int syncs = 0;           // host synchronisations performed by the current call
  int nq = 4;              // Taylor terms per polynomial piece of p(t): 4 (cubic spline) or 12 (node_rule 1)
  int node_rule = 0;       // pexp_options.node_rule
  const int* kprev = nullptr;  // host: Krylov dimension every evaluation needed in the previous WR iteration
  int active_hint = -1;    // evaluations still active in the running EBK loop (-1: unknown);
                           // the profiler's algorithmic byte/flop counts use it
};
extern thread_local CallCfg g_cfg;
// Host synchronisation of the call's stream (counted into pexp_stats.host_syncs).
void host_sync(cudaStream_t st);
// Evaluations a masked launch over E evaluations actually processes (profiler accounting).
inline double eact(int E, const void* active) {
  return (active && g_cfg.active_hint >= 0 && g_cfg.active_hint < E) ? double(g_cfg.active_hint) : double(E);
}

// Tridiagonal rows of the operators A (not M = I - gamma*A): [nops][n] each.
struct Ops {
  int n = 0, nops = 0;
  double *sub = nullptr, *diag = nullptr, *sup = nullptr;
};

// Factorisations of M_f = I - gamma_f A_{op_f}: [nf][n] each.
struct Factors {
  int n = 0, nf = 0, periodic = 0;
  double *l = nullptr, *dinv = nullptr, *sup = nullptr, *z = nullptr, *w = nullptr;
};

// Arguments of the projected-problem kernel (one CTA per evaluation, grid-strided).
struct SPArgs {
  int E, kcap, m, K, kind;       // kind 0: cubic-forced, 1: homogeneous (initial value)
  const double* H;               // [E] ldh x ldh block Hessenberg
  long long hs_e;
  int ldh;
  const int* live;               // [E][ls_e] live flags of basis columns
  long long ls_e;
  const double* gam;             // [E] shift gamma
  double h;                      // piece width
  const int* npieces;            // [E] or nullptr
  int npieces_const;
  int out_stride, nout;          // store z at nodes q*out_stride, q < nout
  const double* coef;            // forced: [E][s-1][nq][m]
  int nq;                        // Taylor terms per piece (4: cubic spline; 12: Chebyshev interpolant pieces)
  int s;
  const double* beta;            // homogeneous: [E] start-vector norms
  const double* crit;            // [E] residual targets
  const double* Gt;              // [E] m x m Gram of (I - gamma A) V_tail
  long long gts_e;
  double* Z;                     // [E][nout][kcap]
  long long zs_e;
  double* res;                   // [E]
  int* conv;                     // [E]
  int* kfin;                     // [E] columns used by the converged z (written on convergence)
  const int* active;             // [E]
  double* work;                  // per-slot workspace (10 Nmax^2)
  long long work_slot;
  int* iwork;
  long long iwork_slot;
  int Nmax;
  int stop_rule;                 // 0: SaI residual ||t||/gamma ; 1: true residual sqrt(t^T Gt t)/gamma
  // kind 2 (grouped homogeneous legs): block 0 = QR of m start vectors, z0 = R0
  const double* R0;              // [E] m x m (ld m)
  const double* critc;           // [E][m] per-leg residual targets
  const int* horc;               // [E][m] per-leg horizons in steps of h (0: unused column)
  int groups;                    // legs of eval e start at j0 = (e % groups) * m
  // exact nested restart (kinds 0/1; DESIGN.md §3 #5).  Completed cycles form the block
  // lower-bidiagonal matrix NA (D x D, compressed coordinates, ld na_ld): diagonal blocks
  // A_hat_c, coupling CPL_c = R_{c+1} TX_c from cycle c into block 0 of cycle c+1.
  double* NA;                    // [E] na_ld x na_ld (nullptr: no restart support)
  int na_ld;
  long long nas_e;
  const int* Dn;                 // [E] nested dimension D
  const int* Kl;                 // [E] compressed width of the last completed cycle
  const double* CPL;             // [E] m x kcap (ld m): coupling rows into the current cycle
  long long cpls_e;
  double* TX;                    // [E] m x kcap (ld m): (1/gamma) H_tail X (written at a restart check)
  int* kplast;                   // [E] compressed width of the current cycle at this check
  int restart_write;             // 1: this check closes a cycle (append to NA, write TX)
};

// Arguments of the fused Arnoldi step (arnoldi.cu), one CTA per evaluation.
struct StepArgs {
  int E, n, m, b, kcap, periodic;
  double* V;
  long long vs_e;
  double* H;                      // ld = kcap
  long long hs_e;
  int* live;                      // [E][kcap]
  const int* fidx;
  const double *fl, *fdinv, *fsup, *fz, *fw;
  double* W0;                     // [E] m x n scratch (raw SaI image)
  long long w0s_e;
  const int* active;
  double defl, piv_tol;
  int rc;
  int cs;                         // CTAs per evaluation (thread-block cluster)
  int ws_smem;                    // 1: the CTA's rows of the new block live in shared memory
  double* hs_g;                   // global scratch for the V^T W partials/sums when they exceed shared memory
  int hs_glob;                    // 1: use hs_g (2 * nv * MB doubles per CTA)
};

// arnoldi.cu
bool arnoldi_fused_ok(int m, int nv, int n, int E, bool have_global_scratch);
size_t arnoldi_scratch_doubles(int E, int kcap, int mcap);
void launch_arnoldi_step(cudaStream_t st, StepArgs a);

// tridiag.cu
void launch_ade_rows(cudaStream_t st, int nops, int n, bool dirichlet, const double* nu, const double* a,
                     double* sub, double* diag, double* sup);
void launch_burgers_rows(cudaStream_t st, int nops, int n, double nu, const double* ubar, double* sub,
                         double* diag, double* sup);
void launch_factor(cudaStream_t st, const Factors& F, int nf, const int* opidx, const double* gam,
                   const Ops& O, int* err);
void launch_sai_solve(cudaStream_t st, const Factors& F, const int* fidx, int E, int ncols,
                      const double* rhs, long long rs_e, int cin0, double* out, long long os_e, int cout0,
                      const int* active, double* out2 = nullptr, long long o2s_e = 0);  // out2: raw copy of x

// tsmm.cu
int xty_chunks(int n, int E);
void xty_tall_plan(int n, int E, int nx, int ny, int& rsub, int& rch, int& nch);
void launch_xty(cudaStream_t st, int E, int n, const double* X, long long xs_e, int x0, int nx,
                const double* Y, long long ys_e, int y0, int ny, double* part, size_t part_cap, double* D,
                long long ds_e, int ldd, int row0, int col0, bool accumulate, const int* active,
                int* cnt = nullptr);
void launch_combine(cudaStream_t st, int E, int n, const double* X, long long xs_e, int x0, int nx,
                    const double* M, long long ms_e, int ldm, double* O, long long os_e, int o0, int ny,
                    double alpha, double beta, const int* active, const int* nxe = nullptr);
void tsmm_init();

// stream.cu: TMA-fed DMMA tall-skinny products of the streaming Arnoldi route
bool stream_ok(int n, int ny);
size_t stream_part_doubles(int E, int n, int nx, int ny);
void launch_sproj(cudaStream_t st, int E, int n, const double* X, long long xs_e, int nx, const double* Y,
                  long long ys_e, int ny, double* part, size_t part_cap, double* D, long long ds_e, int ldd, int row0,
                  int col0, bool accumulate, double* G, long long gs_e, const int* active, int gld = 0,
                  int grow0 = 0, int gcol0 = 0);
void launch_supdate(cudaStream_t st, int E, int n, const double* X, long long xs_e, int nx, const double* M,
                    long long ms_e, int ldm, double* Y, long long ys_e, int ny, double alpha, double beta,
                    const int* active, const int* nxe = nullptr);
void stream_init();

// small.cu
void launch_sym_eig_select(cudaStream_t st, int E, int s, const double* G, double* lam, double* Msel, int* off,
                           double* sigma1, int pass, double tau, double theta, const int* active);
void launch_block_chol(cudaStream_t st, int E, int N, const double* G, long long gs_e, int ldg,
                       const double* norm0, long long ns_e, int ldn, double defl, double* Rinv, const double* Rprev,
                       long long rps_e, int ldrp, double* Rout, long long rs_e, int ldr, int* live,
                       long long ls_e, const int* active, bool pivoted, double dtol = 0.0,
                       double* norm0_out = nullptr, int* maskB = nullptr, int* maskC = nullptr);
void launch_defer_corr(cudaStream_t st, int E, int N, const double* Gb, long long gs_e, const int* cls, long long cs_e,
                       double* Mc, const int* active, bool plus_identity = false);
void launch_onesided_svd(cudaStream_t st, int E, int s, const double* C, const int* kk, double tau, double* Qs,
                         double* sig, double* Cs, int* m_out, const int* active);
void launch_build_final(cudaStream_t st, int E, int s, int mmax, const int* kk, const double* Qs,
                        const double* sig, const double* Cs, const int* m, double* Msel, double* Cfin, int* fill);
void launch_spline(cudaStream_t st, int E, int s, int mmax, const double* Kinv, const double* Cfin, double h,
                   double eta, double* coef, double* crit);
// node_rule 1: coef[e][i][q][c] = sum_k Dmat[i][q][k] Cfin[e][c][k] (Taylor coefficients of the degree-(s-1)
// interpolant through the Chebyshev-Lobatto nodes, at the s-1 uniform piece starts), crit as launch_spline
void launch_poly_coef(cudaStream_t st, int E, int s, int mmax, int nq, const double* Dmat, const double* Cfin,
                      double eta, double* coef, double* crit);
void launch_small_problem(cudaStream_t st, const SPArgs& a, int nslots, int Dmax = 0);
// hom_scan.cu: the Burgers homogeneous scan as one persistent cooperative kernel
bool hom_scan_ok(int n, int kcap);
size_t hom_scan_bytes(int n, int s, int kcap, int P);
int launch_hom_scan(cudaStream_t st, const Factors& F, const double* gam, int P, int s, int n, int kcap, double h,
                    double eta, double defl, const double* u0, const double* Y, const double* Uold, double* Unew,
                    double* delta, char* ws, size_t ws_bytes, int* kscan_rec = nullptr,
                    double* diag = nullptr);  // diag[3] += Arnoldi steps, checks, checker cycles
void launch_restart_finish(cudaStream_t st, int E, int m, int kcap, const double* R, const double* TX, double* CPL,
                           int* Dn, int* Kl, const int* kplast, double* H, long long hs_e, int* live,
                           const int* active);
void launch_small_hom(cudaStream_t st, const SPArgs& a, int nslots);
void launch_expm_batched(cudaStream_t st, int E, int N, const double* A, double* X, double* work,
                         long long work_slot, int* iwork, int nslots);
void small_init();

// stencil.cu: width buckets of the forced EBK (gather into / scatter out of a chunk)
struct GatherArgs {
  const int* perm;
  int wb, mmax, s, n, nq;
  const double *gam, *crit, *coef, *U;
  long long us_e;
  const int *active, *fidx, *opidx;
  double *gam_c, *crit_c, *coef_c, *V;
  long long vs_e;
  int *active_c, *fidx_c, *opidx_c;
};
void launch_bucket_gather(cudaStream_t st, int ec, const GatherArgs& a);
void launch_bucket_scatter(cudaStream_t st, int ec, const int* perm, size_t cnt, const double* Yt, long long yts,
                           double* Y, long long ys_e, const int* krec_c, int* krec);

// stencil.cu
void launch_apply_A(cudaStream_t st, const Ops& O, const int* opidx, int E, int ncols, const double* X,
                    long long xs_e, int x0, double* Y, long long ys_e, int y0, bool periodic);
void launch_apply_M(cudaStream_t st, const Ops& O, const int* opidx, const double* gam, int E, int ncols,
                    const double* X, long long xs_e, int x0, double* Y, long long ys_e, int y0, bool periodic,
                    const int* active);
void launch_lin_source(cudaStream_t st, int batch, int P, int s, int n, const double* Au0, const double* src,
                       double* G);
void launch_fill_random(cudaStream_t st, int E, int n, int mmax, const int* fill, double* V, long long vs_e,
                        unsigned seed);
void launch_broadcast_waveform(cudaStream_t st, int P, int s, int n, const double* u0, double* U);
void launch_ubar_gamma(cudaStream_t st, int P, int s, int n, const double* U, double g0, double* ubar,
                       double* gam);
void launch_burgers_source(cudaStream_t st, int P, int s, int n, double nu, const double* u0, const double* U,
                           const double* ubar, const double* f, double* G);
void launch_wr_step(cudaStream_t st, int s, int n, const double* u0, const double* Wh, const double* Y,
                    const double* Uold, double* Unew, double* uhat_end, double* delta);
void launch_superpose(cudaStream_t st, int batch, int P, int n, const double* u0, const double* Yend,
                      const double* Yh, long long yh_e, long long yh_node, int groups, double* out);
void launch_hom_start_block(cudaStream_t st, int Eh, int mh, int groups, int P, int n, const double* Y, double* V,
                            long long vs_e, double* beta);
void launch_hom_setup_block(cudaStream_t st, int Eh, int mh, int groups, int P, double dT, double eta,
                            const double* beta, double* critc, int* horc, int* active);
void launch_copy_end(cudaStream_t st, int P, int s, int n, const double* U, double* out);
void launch_norms(cudaStream_t st, int E, int n, const double* X, long long xs_e, double* nrm);
void launch_scale_f64(cudaStream_t st, double* y, const double* x, int n, double f);  // y = f x
void launch_scale_cols(cudaStream_t st, int E, int n, const double* X, long long xs_e, const double* nrm,
                       double* Y, long long ys_e);
void launch_add_block(cudaStream_t st, int E, int rows, int cols, const double* S, long long ss_e, int lds,
                      double* D, long long ds_e, int ldd, const int* active);
void launch_hupdate(cudaStream_t st, int E, int rows, int m, const double* T, long long ts_e, int ldt, const double* R,
                    long long rs_e, int ldr, double* H, long long hs_e, int ldh, const int* active);
void launch_hom_setup(cudaStream_t st, int E, int mode, int P, int s, double h, double eta, const double* beta,
                      double* crit, int* npieces, int* active);
void launch_update_active(cudaStream_t st, int E, const int* conv, int* active, int* count, int* krec = nullptr,
                          int kval = 0);
void launch_fill_i32(cudaStream_t st, int* p, int count, int v);
void launch_fill_f64(cudaStream_t st, double* p, size_t count, double v);

}  // namespace pexp
