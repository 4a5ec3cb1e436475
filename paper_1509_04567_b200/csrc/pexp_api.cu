// pexp_api.cu — host orchestration (EBK batch engine, linear Paraexp driver, Burgers WR
// driver) and the C ABI declared in include/pexp.h.  Every arithmetic step runs in the
// CUDA kernels of tridiag.cu / tsmm.cu / small.cu / stencil.cu; this file only sequences
// launches on the caller's stream and carves the caller's workspace.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "pexp.h"

namespace pexp {
thread_local long g_launches = 0;
thread_local CallCfg g_cfg;
bool g_prof_on = false;
// PEXP_SYNC=1: synchronise after every launch to localise a device fault (debugging aid only;
// it changes no numerics, routing or sizes).
bool g_sync_debug = getenv("PEXP_SYNC") != nullptr;

void host_sync(cudaStream_t st) {
  PEXP_CUDA_TRY(cudaStreamSynchronize(st));
  ++g_cfg.syncs;
}
std::vector<ProfRec> g_prof;

// ---------------------------------------------------------------- helper kernels
__global__ void k_set_live0(int E, int kcap, int m, int* live, int keep_block0) {
  const int e = blockIdx.x;
  for (int c = threadIdx.x; c < kcap; c += blockDim.x)
    if (!(keep_block0 && c < m)) live[size_t(e) * kcap + c] = c < m ? 1 : 0;
}

__global__ void k_active_from_m(int E, const int* m, int* active) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) active[e] = m[e] > 0;
}

// Start vectors of the homogeneous legs: eval eh = b*(P-1)+j takes Y[b*P+j] (v_j(T_{j+1})),
// beta = ||.||, Vh block 0 = Y/beta.
__global__ void k_hom_start(int P, int n, const double* Y, long long ys_e, double* beta, double* Vh,
                            long long vs_e) {
  const int eh = blockIdx.x;
  __shared__ double red[32];
  const int b = eh / (P - 1), j = eh % (P - 1);
  const double* y = Y + (long long)(b * P + j) * ys_e;
  double a = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) a = fma(y[r], y[r], a);
  a = sqrt(block_sum(a, red));
  if (threadIdx.x == 0) beta[eh] = a;
  const double sc = a > 0.0 ? 1.0 / a : 0.0;
  double* v = Vh + eh * vs_e;
  for (int r = threadIdx.x; r < n; r += blockDim.x) v[r] = y[r] * sc;
}

static void check_err(cudaStream_t st) { PEXP_CUDA_TRY(cudaGetLastError()); (void)st; }

template <class T>
static void h2d(cudaStream_t st, T* dst, const std::vector<T>& v) {
  if (v.empty()) return;
  PEXP_CUDA_TRY(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  host_sync(st);  // pageable source: keep it alive until copied
}

// ---------------------------------------------------------------- options
// node_rule 1: p(t) = the degree-(s-1) interpolant through the Chebyshev-Lobatto
// nodes, integrated through its Taylor polynomials of NQ_CHEB terms on the s-1 uniform pieces
constexpr int NQ_CHEB = 12;
struct Opts {
  int s;
  double tau_f, eta_f;
  int restart_blocks, kcap, stop_rule, kcyc, chunk, nq, node_rule;
  cudaStream_t st;
  CallCfg cfg;
};

static Opts norm_opts(const pexp_options& o) {
  Opts r;
  r.s = o.s > 0 ? o.s : 32;
  r.tau_f = o.svd_tau_factor > 0 ? o.svd_tau_factor : 0.01;
  r.eta_f = o.stop_factor > 0 ? o.stop_factor : 0.1;
  r.restart_blocks = o.restart_blocks > 0 ? o.restart_blocks : (o.restart_blocks < 0 ? 0 : 20);
  r.kcap = o.k_max > 0 ? o.k_max : 256;
  r.kcyc = o.basis_cols > 0 ? std::min(o.basis_cols, r.kcap) : r.kcap;
  r.chunk = o.eval_chunk > 0 ? o.eval_chunk : (1 << 30);
  r.st = (cudaStream_t)o.stream;
  r.stop_rule = o.stop_rule;
  r.cfg.defl = o.defl_tol > 0 ? o.defl_tol : 1e-10;
  r.cfg.piv_tol = o.piv_tol > 0 ? o.piv_tol : 1e-14;
  r.cfg.route = o.route;
  r.cfg.hom_group = o.hom_group > 0 ? std::min(o.hom_group, 16) : 8;
  r.cfg.buckets = o.width_buckets >= 0 ? 1 : 0;
  r.cfg.syncs = 0;
  r.node_rule = o.node_rule;
  r.nq = o.node_rule == 1 ? NQ_CHEB : 4;
  r.cfg.nq = r.nq;
  r.cfg.node_rule = r.node_rule;
  return r;
}

// ---------------------------------------------------------------- EBK buffers
struct EbkBufs {
  int E = 0, n = 0, kcap = 0, ktot = 0, mcap = 0, nout = 0, s = 0, groups = 1, nq = 4;
  long long vs_e = 0, hs_e = 0, zs_e = 0;
  double *V, *H, *Z, *Gt, *Wt, *Wt2, *T, *G0, *G1, *Rinv, *Rtmp, *res, *gam, *crit, *beta, *coef, *n0p, *R0, *critc;
  int *live, *active, *conv, *kfin, *npieces, *count, *fidx, *opidx, *xcnt, *horc, *krec;
  int *maskB, *maskC;  // in-block QR: evaluations that need stage B / stage C (written by k_block_chol)
  double* part;
  size_t part_cap;
  double* stepws = nullptr;  // fused Arnoldi step: global V^T W partials (large bases)
  double* spart = nullptr;   // streaming route: per-chunk partials of [V W]^T W
  size_t spart_cap = 0;
  // width buckets of the forced EBK (ebk_forced_bucketed): permutation [E] and the chunk-slot
  // copies of the per-evaluation inputs / outputs (nullptr: bucketing not planned)
  int* perm = nullptr;
  double *gam_c = nullptr, *crit_c = nullptr, *coef_c = nullptr, *Ytmp = nullptr;
  int *active_c = nullptr, *fidx_c = nullptr, *opidx_c = nullptr, *krec_c = nullptr;
  int ycols = 0;
  double* work;
  int* iwork;
  int nslots, Nmax;
  long long work_slot, iwork_slot;
  // exact nested restart (nullptr when the run cannot restart)
  double *NA = nullptr, *CPL = nullptr, *TX = nullptr;
  int *Dn = nullptr, *Kl = nullptr, *kplast = nullptr;
};

// xty partial-sum capacity for E evaluations of an (nx x ny) product (see launch_xty)
static size_t part_need(int E, int n, int nx, int ny) {
  // bound on E'*nch(E') for every E' <= E (xty_chunks stops at <= 1184 CTAs or one chunk)
  size_t ech = std::max<size_t>(size_t(E) * cdiv(n, xty_chunks(n, E)), 2 * 148 * 8 + size_t(E));
  ech = std::min<size_t>(ech, size_t(E) * cdiv(n, 512));
  size_t cap = ech * nx * ny;
  // tall path (ny <= 32): E' * nch(E') <= E' + 2*148*6 chunks for any E' <= E
  size_t tall = (size_t(E) + 2 * 148 * 6) * size_t(nx) * std::min(ny, 32);
  return std::max(cap, tall);
}

// E evaluations run through the EBK in chunks of at most Ec (eval_chunk option): the light
// per-evaluation arrays (inputs set by the SVD stage / callers, flags, residuals) cover all E,
// the basis and everything else that scales with the Krylov dimension covers one chunk.
// kcap: basis columns per evaluation and cycle; ktot: total Krylov dimension over all cycles
// (ktot > kcap or restart_blocks > 0 allocates the nested-restart state).
static void alloc_ebk(Arena& ar, EbkBufs& B, int E, int Ec, int n, int kcap, int ktot, int mcap, int nout, int s,
                      bool forced, double* Wt_shared, bool restartable, int ycols = 0, int nq = 4) {
  Ec = std::max(1, std::min(E, Ec));
  B.nq = nq;
  B.E = Ec; B.n = n; B.kcap = kcap; B.ktot = ktot; B.mcap = mcap; B.nout = nout; B.s = s;
  B.vs_e = (long long)kcap * n;
  B.hs_e = (long long)kcap * kcap;
  B.zs_e = (long long)nout * kcap;
  // ---- light, all evaluations
  B.res = ar.take<double>(E);
  B.gam = ar.take<double>(E);
  B.crit = ar.take<double>(E);
  B.beta = ar.take<double>(size_t(E) * mcap);
  B.coef = forced ? ar.take<double>(size_t(E) * (s - 1) * nq * mcap) : nullptr;
  B.active = ar.take<int>(E);
  B.conv = ar.take<int>(E);
  B.kfin = ar.take<int>(E);
  B.npieces = ar.take<int>(E);
  B.count = ar.take<int>(4);
  B.fidx = ar.take<int>(E);
  B.opidx = ar.take<int>(E);
  B.xcnt = ar.take<int>(E);
  B.krec = ar.take<int>(E);
  // ---- heavy, one chunk
  B.V = ar.take<double>(size_t(Ec) * kcap * n);
  B.H = ar.take<double>(size_t(Ec) * kcap * kcap);
  B.Z = ar.take<double>(size_t(Ec) * nout * kcap);
  B.Gt = ar.take<double>(size_t(Ec) * mcap * mcap);
  B.Wt = Wt_shared ? Wt_shared : ar.take<double>(size_t(Ec) * mcap * n);
  B.Wt2 = ar.take<double>(size_t(Ec) * mcap * n);
  B.n0p = ar.take<double>(size_t(Ec) * mcap);
  B.T = ar.take<double>(size_t(Ec) * kcap * mcap);
  B.G0 = ar.take<double>(size_t(Ec) * mcap * mcap);
  B.G1 = ar.take<double>(size_t(Ec) * mcap * mcap);
  B.Rinv = ar.take<double>(size_t(Ec) * mcap * mcap);
  B.Rtmp = ar.take<double>(size_t(Ec) * mcap * mcap);
  B.R0 = ar.take<double>(size_t(Ec) * mcap * mcap);
  B.critc = ar.take<double>(size_t(Ec) * mcap);
  B.horc = ar.take<int>(size_t(Ec) * mcap);
  B.live = ar.take<int>(size_t(Ec) * kcap);
  B.maskB = ar.take<int>(Ec);
  B.maskC = ar.take<int>(Ec);
  // the SVD stage (all E, s x s products) shares the partial-sum buffer with the chunks
  B.part_cap = std::max(part_need(Ec, n, std::max(kcap, s), forced ? std::max(mcap, s) : mcap),
                        forced ? part_need(E, n, s, s) : size_t(0));
  if (forced && stream_ok(n, 32))  // SVD-stage products with up to s columns through the streaming kernels
    B.part_cap = std::max(B.part_cap, stream_part_doubles(E, n, s, std::min(s, 32)));
  B.part = ar.take<double>(B.part_cap);
  {
    const size_t sw = arnoldi_scratch_doubles(Ec, kcap, mcap);
    B.stepws = sw ? ar.take<double>(sw) : nullptr;
  }
  if (stream_ok(n, std::min(mcap, 32))) {
    B.spart_cap = stream_part_doubles(Ec, n, kcap + std::min(mcap, 32), std::min(mcap, 32));
    B.spart = ar.take<double>(B.spart_cap);
  }
  B.Nmax = ktot + (forced ? nq * mcap : 0);
  B.work_slot = 10LL * B.Nmax * B.Nmax;
  B.iwork_slot = B.Nmax;
  // one workspace slot per resident cluster; large projected problems get one per SM
  B.nslots = std::min(Ec, B.Nmax > 512 ? 148 : 512);
  B.work = ar.take<double>(size_t(B.nslots) * B.work_slot);
  B.iwork = ar.take<int>(size_t(B.nslots) * B.iwork_slot);
  if (forced && ycols > 0 && E > 1) {  // width buckets
    B.ycols = ycols;
    B.perm = ar.take<int>(E);
    B.gam_c = ar.take<double>(Ec);
    B.crit_c = ar.take<double>(Ec);
    B.active_c = ar.take<int>(Ec);
    B.fidx_c = ar.take<int>(Ec);
    B.opidx_c = ar.take<int>(Ec);
    B.krec_c = ar.take<int>(Ec);
    B.coef_c = ar.take<double>(size_t(Ec) * (s - 1) * nq * mcap);
    B.Ytmp = ar.take<double>(size_t(Ec) * ycols * n);
  }
  if (restartable) {
    B.NA = ar.take<double>(size_t(Ec) * ktot * ktot);
    B.CPL = ar.take<double>(size_t(Ec) * mcap * kcap);
    B.TX = ar.take<double>(size_t(Ec) * mcap * kcap);
    B.Dn = ar.take<int>(Ec);
    B.Kl = ar.take<int>(Ec);
    B.kplast = ar.take<int>(Ec);
  }
}

// View of evaluations [c0, c0 + Ec) of B for one EBK chunk (light arrays offset, heavy shared).
static EbkBufs chunk_view(const EbkBufs& B, int c0, int Ec, int mb) {
  EbkBufs C = B;
  C.E = Ec;
  C.res += c0; C.gam += c0; C.crit += c0; C.active += c0; C.conv += c0; C.kfin += c0;
  C.npieces += c0; C.fidx += c0; C.opidx += c0; C.xcnt += c0; C.krec += c0;
  C.beta += c0;  // kind-1 layout (forced chunks do not read beta)
  if (C.coef) C.coef += size_t(c0) * (B.s - 1) * B.nq * mb;
  return C;
}

// Pivoted deflating Cholesky-QR of the m columns of V at column offset c0 (in place):
// Gram -> k_block_chol -> W <- W Rinv.  norm0 (nullable) = pre-orthogonalisation norms for
// the deflation test; dtol > 0 defers nearly dependent columns (class 2, passed through raw).
static void chol_combine_block(cudaStream_t st, EbkBufs& B, int E, int n, int m, int c0, const double* n0,
                               long long n0s, int n0ld, double dtol, double defl, double* n0out, const int* active,
                               bool masks = false) {
  const long long ws_e = B.vs_e;
  launch_xty(st, E, n, B.V, ws_e, c0, m, B.V, ws_e, c0, m, B.part, B.part_cap, B.G1, (long long)m * m, m, 0, 0, false,
             active, B.xcnt);
  launch_block_chol(st, E, m, B.G1, (long long)m * m, m, n0, n0s, n0ld, defl, B.Rinv, nullptr, 0, 0, nullptr, 0, 0,
                    B.live + c0, B.kcap, active, true, dtol, n0out, masks ? B.maskB : nullptr,
                    masks ? B.maskC : nullptr);
  if (m <= 32) {
    launch_combine(st, E, n, B.V, ws_e, c0, m, B.Rinv, (long long)m * m, m, B.V, ws_e, c0, m, 1.0, 0.0, active);
  } else {
    launch_combine(st, E, n, B.V, ws_e, c0, m, B.Rinv, (long long)m * m, m, B.Wt2, (long long)m * n, 0, m, 1.0, 0.0,
                   active);
    PEXP_CUDA_TRY(cudaMemcpy2DAsync(B.V + size_t(c0) * n, ws_e * sizeof(double), B.Wt2, size_t(m) * n * sizeof(double),
                                    size_t(m) * n * sizeof(double), E, cudaMemcpyDeviceToDevice, st));
  }
}

// Robust in-block QR of the m columns at offset c0 (already orthogonal to earlier columns up to
// the first BCGS pass): stage A accepts well-separated columns (scaled pivot > 1e-8), defers
// nearly dependent ones; stage B re-orthogonalises deferred columns explicitly (CGS2); stage C
// accepts or deflates them relative to their pre-orthogonalisation norms norm0.
// Stage B runs only for the evaluations whose stage A deferred a column (device-side mask written
// by k_block_chol: the other evaluations' work items exit at once).  With reorth_follows (the call
// inside an Arnoldi step, where BCGS pass 2 and its CholQR follow) stage C is likewise masked to
// the evaluations whose stage A did not accept every column with scaled pivots >= 1e-2 -- the rule
// of the fused step (arnoldi.cu).  The masked launches are charged no algorithmic bytes.
static void inblock_qr(cudaStream_t st, EbkBufs& B, int E, int n, int m, int c0, const double* norm0, long long n0s,
                       int n0ld, double defl, const int* active, bool reorth_follows = false) {
  const long long ws_e = B.vs_e;
  const int* act0 = active;
  chol_combine_block(st, B, E, n, m, c0, norm0, n0s, n0ld, 1e-8, defl, B.n0p, active, true);
  // (wide blocks m > 32 go out of place through Wt2 and copy every evaluation back: no masks there)
  const bool mask_ok = m <= 32;
  const int hint = g_cfg.active_hint;
  if (mask_ok) {
    g_cfg.active_hint = 0;
    active = B.maskB;
  }
  for (int rep = 0; rep < 2; ++rep) {
    launch_xty(st, E, n, B.V, ws_e, c0, m, B.V, ws_e, c0, m, B.part, B.part_cap, B.G1, (long long)m * m, m, 0, 0, false,
               active, B.xcnt);
    if (m <= 32) {
      launch_defer_corr(st, E, m, B.G1, (long long)m * m, B.live + c0, B.kcap, B.Rinv, active);
      launch_combine(st, E, n, B.V, ws_e, c0, m, B.Rinv, (long long)m * m, m, B.V, ws_e, c0, m, 1.0, 1.0, active);
    } else {  // wider blocks: V_blk (I + Mc) out of place, then copied back
      launch_defer_corr(st, E, m, B.G1, (long long)m * m, B.live + c0, B.kcap, B.Rinv, active, true);
      launch_combine(st, E, n, B.V, ws_e, c0, m, B.Rinv, (long long)m * m, m, B.Wt2, (long long)m * n, 0, m, 1.0, 0.0,
                     active);
      PEXP_CUDA_TRY(cudaMemcpy2DAsync(B.V + size_t(c0) * n, ws_e * sizeof(double), B.Wt2,
                                      size_t(m) * n * sizeof(double), size_t(m) * n * sizeof(double), E,
                                      cudaMemcpyDeviceToDevice, st));
    }
  }
  const bool maskc = mask_ok && reorth_follows;
  if (!maskc) g_cfg.active_hint = hint;
  chol_combine_block(st, B, E, n, m, c0, B.n0p, m, 0, 0.0, defl, nullptr, maskc ? B.maskC : act0);
  g_cfg.active_hint = hint;
}

struct RunInfo {
  int max_k = 0;     // largest basis width of a cycle (columns of V to combine)
  int max_ktot = 0;  // largest total Krylov dimension over the cycles
  int restarts = 0;
  int unconverged = 0;
  double worst_res_ratio = 0.0;
  int chunks = 0, buckets = 1;
};

// Where a restart accumulates the outputs of a closed cycle: Y[e*ys_e + j*n] += V_c z_c at
// output o0 + j, j < no.  The caller's final combine then adds (beta = 1) when restarts > 0.
struct Accum {
  double* Y = nullptr;
  long long ys_e = 0;
  int o0 = 0, no = 0;
};

// SaI block Arnoldi with BCGS2 + deflating CholQR2, projected problem checks on a geometric
// schedule.  Preconditions: V block 0 (m columns) orthonormal; active, gam, fidx, opidx set;
// forced: coef and crit set; homogeneous: beta, crit, npieces set.
static RunInfo ebk_run(cudaStream_t st, EbkBufs& B, const Factors& F, const Ops& O, bool periodic, int m,
                       int kind, double h, int npieces_const, int out_stride, int nout, int stop_rule,
                       Accum acc = Accum{}, int restart_blocks = 0, int first_hint = 0) {
  RunInfo info;
  const int E = B.E, n = B.n, kcap = B.kcap;
  if (E == 0) return info;
  if (m > B.mcap) fail(1, "block width exceeds capacity");
  PEXP_CUDA_TRY(cudaMemsetAsync(B.xcnt, 0, E * sizeof(int), st));
  k_set_live0<<<E, 128, 0, st>>>(E, kcap, m, B.live, kind == 2 ? 1 : 0);
  count_launch();
  launch_fill_f64(st, B.H, size_t(E) * kcap * kcap, 0.0);
  launch_fill_f64(st, B.Z, size_t(E) * nout * kcap, 0.0);
  launch_fill_i32(st, B.kfin, E, 0);
  launch_fill_i32(st, B.conv, E, 0);
  PEXP_LAUNCH_CHECK();
  // fused cluster step (arnoldi.cu) whenever the step's panels fit shared memory
  int steps = 0, last_check = -1;
  int next_check = std::max(4, 2 * m);
  // WR iterations after the first: no evaluation of this run converged below first_hint columns last
  // time, so the checks before ~0.8 first_hint are skipped (the operators change little between iterations)
  if (first_hint > 0) next_check = std::max(next_check, std::min(int(0.8 * first_hint) / m * m, kcap - 2 * m));
  // deflation: a new column is dropped when BCGS leaves < defl (default 1e-10) of
  // ||(I - gamma A)^{-1} v|| (well above the shift-and-invert solve rounding (~1e-13..1e-12),
  // below the 1e-8 parity bar); pexp_options.defl_tol
  const double defl = g_cfg.defl;
  SPArgs a{};
  a.E = E; a.kcap = kcap; a.m = m; a.kind = kind;
  a.H = B.H; a.hs_e = B.hs_e; a.ldh = kcap;
  a.live = B.live; a.ls_e = kcap;
  a.gam = B.gam; a.h = h;
  a.npieces = kind == 1 ? B.npieces : nullptr;
  a.npieces_const = npieces_const;
  a.out_stride = out_stride; a.nout = nout;
  a.coef = B.coef; a.s = B.s; a.nq = B.nq;
  a.beta = B.beta; a.crit = B.crit;
  a.Gt = B.Gt; a.gts_e = (long long)m * m;
  a.Z = B.Z; a.zs_e = B.zs_e;
  a.res = B.res; a.conv = B.conv; a.kfin = B.kfin; a.active = B.active;
  a.work = B.work; a.work_slot = B.work_slot; a.iwork = B.iwork; a.iwork_slot = B.iwork_slot; a.Nmax = B.Nmax;
  a.stop_rule = stop_rule;
  a.R0 = B.R0; a.critc = B.critc; a.horc = B.horc; a.groups = std::max(1, B.groups);
  const bool can_restart = kind != 2 && acc.Y != nullptr && B.NA != nullptr;
  if (can_restart) {
    a.NA = B.NA; a.na_ld = B.ktot; a.nas_e = (long long)B.ktot * B.ktot;
    a.Dn = B.Dn; a.Kl = B.Kl; a.CPL = B.CPL; a.cpls_e = (long long)m * kcap;
    a.TX = B.TX; a.kplast = B.kplast;
    launch_fill_i32(st, B.Dn, E, 0);
    launch_fill_i32(st, B.Kl, E, 0);
    launch_fill_f64(st, B.NA, size_t(E) * B.ktot * B.ktot, 0.0);  // blocks above/below the bidiagonal
  }
  int Koff = 0;  // columns (uncompressed) of the closed cycles
  int remaining = E;
  std::vector<double> prevq(E, -1.0), curq(E, -1.0);
  std::vector<int> prevK(E, -1);
  std::vector<double> hres(E), hcrit(E);
  std::vector<int> hact(E);
  int predicted_next = -1;
  auto do_check = [&](int K, bool closing) {
    if (stop_rule == 1) {  // true residual: tail Gram of Wt = (I - gamma A) V[:, K:K+m]
      launch_apply_M(st, O, B.opidx, B.gam, E, m, B.V, B.vs_e, K, B.Wt, (long long)m * n, 0, periodic, B.active);
      launch_xty(st, E, n, B.Wt, (long long)m * n, 0, m, B.Wt, (long long)m * n, 0, m, B.part, B.part_cap, B.Gt,
                 (long long)m * m, m, 0, 0, false, B.active, B.xcnt);
    }
    a.K = K;
    a.restart_write = closing ? 1 : 0;
    if (Koff + K > B.ktot) fail(1, "small problem exceeds workspace");
    if (kind == 2)
      launch_small_hom(st, a, B.nslots);
    else
      launch_small_problem(st, a, B.nslots, Koff);
    PEXP_CUDA_TRY(cudaMemsetAsync(B.count, 0, sizeof(int), st));
    launch_update_active(st, E, B.conv, B.active, B.count, B.krec, Koff + K);
    // one synchronisation per check: the active count and the residual ratios that place the next check
    int h_count = 0;
    PEXP_CUDA_TRY(cudaMemcpyAsync(&h_count, B.count, sizeof(int), cudaMemcpyDeviceToHost, st));
    PEXP_CUDA_TRY(cudaMemcpyAsync(hres.data(), B.res, E * sizeof(double), cudaMemcpyDeviceToHost, st));
    PEXP_CUDA_TRY(cudaMemcpyAsync(hcrit.data(), B.crit, E * sizeof(double), cudaMemcpyDeviceToHost, st));
    PEXP_CUDA_TRY(cudaMemcpyAsync(hact.data(), B.active, E * sizeof(int), cudaMemcpyDeviceToHost, st));
    host_sync(st);
    remaining = h_count;
    g_cfg.active_hint = remaining;
    last_check = K;
    info.max_k = std::max(info.max_k, K);
    info.max_ktot = std::max(info.max_ktot, Koff + K);
    const int Kt = Koff + K;  // the residual decays with the total dimension
    // predict the K at which the still-active evaluations converge: the residual ratio
    // q = res/crit decays roughly geometrically in K; extrapolate from the last two checks
    predicted_next = -1;
    if (remaining > 0) {
      std::vector<double> preds;
      for (int e = 0; e < E; ++e) {
        if (!hact[e] || !(kind == 2 || hcrit[e] > 0)) continue;
        double q = kind == 2 ? hres[e] : hres[e] / hcrit[e];
        if (prevK[e] >= 0 && prevK[e] < Kt && prevq[e] > 0 && q > 0 && q < prevq[e]) {
          double slope = (std::log(q) - std::log(prevq[e])) / double(Kt - prevK[e]);
          preds.push_back(Kt + std::log(0.5 / q) / slope - Koff);
        }
        prevq[e] = q;
        prevK[e] = Kt;
      }
      if (!preds.empty()) {
        std::sort(preds.begin(), preds.end());
        double p80 = preds[std::min(preds.size() - 1, size_t(0.8 * preds.size()))];
        predicted_next = (int)std::ceil(p80);
      }
    }
  };
  // initial active count (some evals may start inactive: zero source / zero start vector)
  {
    PEXP_CUDA_TRY(cudaMemsetAsync(B.count, 0, sizeof(int), st));
    launch_update_active(st, E, B.conv, B.active, B.count);
    int h_count = 0;
    PEXP_CUDA_TRY(cudaMemcpyAsync(&h_count, B.count, sizeof(int), cudaMemcpyDeviceToHost, st));
    host_sync(st);
    remaining = h_count;
    g_cfg.active_hint = remaining;
  }
  while (remaining > 0) {
    const bool cyc_full = (steps + 2) * m > kcap;            // no room for another block + tail
    const bool tot_full = Koff + (steps + 1) * m > B.ktot;    // total dimension cap
    const bool count_hit = can_restart && restart_blocks > 0 && steps >= restart_blocks;
    if (tot_full || (cyc_full && !can_restart)) {
      if (steps >= 1 && last_check != steps * m) do_check(steps * m, false);
      break;
    }
    if (cyc_full || count_hit) {
      if (steps == 0) fail(1, "basis capacity below two blocks");
      // ---- exact nested restart (DESIGN.md §3 #5): close cycle c at K = steps*m
      const int K = steps * m;
      do_check(K, true);  // z at the outputs, NA extended by this cycle, TX = H_tail X / gamma
      if (remaining == 0) break;
      const long long ws_e = B.vs_e;
      if (info.restarts == 0)
        PEXP_CUDA_TRY(cudaMemsetAsync(acc.Y, 0, size_t(E) * acc.ys_e * sizeof(double), st));
      // outputs of the closed cycle: Y += V_c z_c
      launch_combine(st, E, n, B.V, ws_e, 0, K, B.Z + size_t(acc.o0) * kcap, B.zs_e, kcap, acc.Y, acc.ys_e, 0,
                     acc.no, 1.0, 1.0, B.active);
      // residual r(t) = (1/gamma) W TX z(t),  W = (I - gamma A) V_tail  ->  new block 0 = Q, W = Q R
      launch_apply_M(st, O, B.opidx, B.gam, E, m, B.V, ws_e, K, B.V, ws_e, 0, periodic, B.active);
      PEXP_CUDA_TRY(cudaMemcpy2DAsync(B.Wt, size_t(m) * n * sizeof(double), B.V, ws_e * sizeof(double),
                                      size_t(m) * n * sizeof(double), E, cudaMemcpyDeviceToDevice, st));
      launch_xty(st, E, n, B.V, ws_e, 0, m, B.V, ws_e, 0, m, B.part, B.part_cap, B.G0, (long long)m * m, m, 0, 0,
                 false, B.active, B.xcnt);
      inblock_qr(st, B, E, n, m, 0, B.G0, (long long)m * m, m, defl, B.active);
      launch_xty(st, E, n, B.V, ws_e, 0, m, B.Wt, (long long)m * n, 0, m, B.part, B.part_cap, B.Rtmp,
                 (long long)m * m, m, 0, 0, false, B.active, B.xcnt);
      launch_restart_finish(st, E, m, kcap, B.Rtmp, B.TX, B.CPL, B.Dn, B.Kl, B.kplast, B.H, B.hs_e, B.live,
                            B.active);
      Koff += K;
      ++info.restarts;
      steps = 0;
      last_check = -1;
      next_check = std::max(4, 2 * m);
      if (predicted_next > 0) next_check = std::max(m, std::min(predicted_next - K, kcap));
      continue;
    }
    const int b = steps, nv = (b + 1) * m;
    const long long ws_e = B.vs_e;
    if (g_cfg.route != 1 && arnoldi_fused_ok(m, nv, n, E, B.stepws != nullptr)) {  // one cluster per evaluation: whole step
      StepArgs sa{};
      sa.E = E; sa.n = n; sa.m = m; sa.b = b; sa.kcap = kcap; sa.periodic = F.periodic;
      sa.V = B.V; sa.vs_e = B.vs_e; sa.H = B.H; sa.hs_e = B.hs_e; sa.live = B.live; sa.fidx = B.fidx;
      sa.fl = F.l; sa.fdinv = F.dinv; sa.fsup = F.sup; sa.fz = F.z; sa.fw = F.w;
      sa.W0 = B.Wt; sa.w0s_e = (long long)m * n; sa.active = B.active; sa.defl = defl;
      sa.hs_g = B.stepws;
      launch_arnoldi_step(st, sa);
    } else if (B.spart && m <= 32) {  // streaming route: TMA-fed DMMA products (stream.cu)
    // W0 = (I - gamma A)^{-1} V_b into the basis (columns [nv, nv+m)) and, raw, into Wt
    launch_sai_solve(st, F, B.fidx, E, m, B.V, ws_e, b * m, B.V, ws_e, nv, B.active, B.Wt, (long long)m * n);
    // BCGS pass 1: H[0:nv, block b] = V^T W0 and the W0 Gram (deflation reference) in one pass
    launch_sproj(st, E, n, B.V, ws_e, nv, B.V + size_t(nv) * n, ws_e, m, B.spart, B.spart_cap, B.H, B.hs_e, kcap, 0,
                 b * m, false, B.G0, (long long)m * m, B.active);
    launch_supdate(st, E, n, B.V, ws_e, nv, B.H + size_t(b) * m * kcap, B.hs_e, kcap, B.V + size_t(nv) * n, ws_e, m,
                   -1.0, 1.0, B.active);
    inblock_qr(st, B, E, n, m, nv, B.G0, (long long)m * m, m, defl, B.active, true);
    // BCGS pass 2 + CholQR
    launch_sproj(st, E, n, B.V, ws_e, nv, B.V + size_t(nv) * n, ws_e, m, B.spart, B.spart_cap, B.T,
                 (long long)kcap * B.mcap, nv, 0, 0, false, nullptr, 0, B.active);
    launch_supdate(st, E, n, B.V, ws_e, nv, B.T, (long long)kcap * B.mcap, nv, B.V + size_t(nv) * n, ws_e, m, -1.0,
                   1.0, B.active);
    chol_combine_block(st, B, E, n, m, nv, nullptr, 0, 0, 0.0, defl, nullptr, B.active);
    launch_xty(st, E, n, B.V, ws_e, nv, m, B.Wt, (long long)m * n, 0, m, B.part, B.part_cap, B.H, B.hs_e, kcap, nv,
               b * m, false, B.active, B.xcnt);
    } else {
    // W = (I - gamma A)^{-1} V_b  -> columns [nv, nv+m)
    // keep the raw image W0 = (I - gamma A)^{-1} V_b (second output Wt): the subdiagonal block of H
    // is computed directly as Q^T W0 at the end (exact to eps, independent of the in-block QR route)
    launch_sai_solve(st, F, B.fidx, E, m, B.V, ws_e, b * m, B.V, ws_e, nv, B.active, B.Wt, (long long)m * n);
    // norms of W0 (deflation reference)
    launch_xty(st, E, n, B.V, ws_e, nv, m, B.V, ws_e, nv, m, B.part, B.part_cap, B.G0, (long long)m * m, m, 0, 0,
               false, B.active, B.xcnt);
    // BCGS pass 1: H[0:nv, block b] = V^T W0 ; W = W0 - V H
    launch_xty(st, E, n, B.V, ws_e, 0, nv, B.V, ws_e, nv, m, B.part, B.part_cap, B.H, B.hs_e, kcap, 0, b * m,
               false, B.active, B.xcnt);
    launch_combine(st, E, n, B.V, ws_e, 0, nv, B.H + size_t(b) * m * kcap, B.hs_e, kcap, B.V, ws_e, nv, m, -1.0, 1.0,
                   B.active);
    inblock_qr(st, B, E, n, m, nv, B.G0, (long long)m * m, m, defl, B.active, true);
    // BCGS pass 2 (re-orthogonalisation against V) + CholQR of the nearly orthonormal block
    launch_xty(st, E, n, B.V, ws_e, 0, nv, B.V, ws_e, nv, m, B.part, B.part_cap, B.T, (long long)kcap * B.mcap, nv,
               0, 0, false, B.active, B.xcnt);
    launch_combine(st, E, n, B.V, ws_e, 0, nv, B.T, (long long)kcap * B.mcap, nv, B.V, ws_e, nv, m, -1.0, 1.0,
                   B.active);
    chol_combine_block(st, B, E, n, m, nv, nullptr, 0, 0, 0.0, defl, nullptr, B.active);
    // subdiagonal block: H[nv:nv+m, block b] = Q^T W0
    launch_xty(st, E, n, B.V, ws_e, nv, m, B.Wt, (long long)m * n, 0, m, B.part, B.part_cap, B.H, B.hs_e, kcap, nv,
               b * m, false, B.active, B.xcnt);
    }
    ++steps;
    const int K = steps * m;
    const bool closing_next = (steps + 2) * m > kcap || Koff + (steps + 1) * m > B.ktot ||
                              (can_restart && restart_blocks > 0 && steps >= restart_blocks);
    if (!(closing_next && can_restart) && (K >= next_check || closing_next)) {
      do_check(K, false);
      int geo = std::max(K + m, (int)std::ceil(K * 1.25));
      next_check = geo;
      if (predicted_next > 0) next_check = std::max(K + m, std::min(predicted_next, 2 * K));
    }
  }
  info.unconverged = remaining;
  g_cfg.active_hint = -1;
  // worst residual / target over the evaluations at their last check (diagnostic; the host copies of
  // the last check)
  for (int e = 0; e < E; ++e)
    if (last_check >= 0 && (kind == 2 || hcrit[e] > 0))
      info.worst_res_ratio = std::max(info.worst_res_ratio, kind == 2 ? hres[e] : hres[e] / hcrit[e]);
  return info;
}

// ---------------------------------------------------------------- source SVD stage
struct SvdBufs {
  double *U, *R, *Gs, *lam, *Msel, *sigma1, *Cb, *Qs, *Cs, *sig, *Cfin, *Rinv, *Kinv, *Dmat;
  int *off, *me, *fill;
  bool pt_ready = false;  // the p(t) matrix (Kinv / Dmat) is on the device for this solve
};

static void alloc_svd(Arena& ar, SvdBufs& S, int E, int n, int s) {
  S.U = ar.take<double>(size_t(E) * s * n);
  S.R = ar.take<double>(size_t(E) * s * n);
  S.Gs = ar.take<double>(size_t(E) * s * s);
  S.lam = ar.take<double>(size_t(E) * s);
  S.Msel = ar.take<double>(size_t(E) * s * s);
  S.sigma1 = ar.take<double>(E);
  S.Cb = ar.take<double>(size_t(E) * s * s);
  S.Qs = ar.take<double>(size_t(E) * s * s);
  S.Cs = ar.take<double>(size_t(E) * s * s);
  S.sig = ar.take<double>(size_t(E) * s);
  S.Cfin = ar.take<double>(size_t(E) * s * s);
  S.Rinv = ar.take<double>(size_t(E) * s * s);
  S.Kinv = ar.take<double>(size_t(s) * s);
  S.Dmat = ar.take<double>(size_t(s - 1) * NQ_CHEB * s);
  S.off = ar.take<int>(E);
  S.me = ar.take<int>(E);
  S.fill = ar.take<int>(size_t(E) * s);
}

// Not-a-knot system matrix (rows: M0-2M1+M2 = 0; M_{i-1}+4M_i+M_{i+1} = r_i; last analogous),
// inverted on the host once per solve (depends on s only).
static std::vector<double> notaknot_inverse(int s) {
  std::vector<double> K(size_t(s) * s, 0.0), I(size_t(s) * s, 0.0);
  auto at = [&](std::vector<double>& M, int i, int j) -> double& { return M[i + size_t(j) * s]; };
  at(K, 0, 0) = 1; at(K, 0, 1) = -2; at(K, 0, 2) = 1;
  at(K, s - 1, s - 3) = 1; at(K, s - 1, s - 2) = -2; at(K, s - 1, s - 1) = 1;
  for (int i = 1; i < s - 1; ++i) { at(K, i, i - 1) = 1; at(K, i, i) = 4; at(K, i, i + 1) = 1; }
  for (int i = 0; i < s; ++i) at(I, i, i) = 1;
  // Gauss-Jordan with partial pivoting
  for (int c = 0; c < s; ++c) {
    int p = c;
    for (int r = c + 1; r < s; ++r) if (std::fabs(at(K, r, c)) > std::fabs(at(K, p, c))) p = r;
    if (p != c) for (int j = 0; j < s; ++j) { std::swap(at(K, c, j), at(K, p, j)); std::swap(at(I, c, j), at(I, p, j)); }
    double d = at(K, c, c);
    for (int j = 0; j < s; ++j) { at(K, c, j) /= d; at(I, c, j) /= d; }
    for (int r = 0; r < s; ++r)
      if (r != c) {
        double f = at(K, r, c);
        if (f != 0.0) for (int j = 0; j < s; ++j) { at(K, r, j) -= f * at(K, c, j); at(I, r, j) -= f * at(I, c, j); }
      }
  }
  return I;
}

// node_rule 1 ("Chebyshev nodes", "other types of p(t) possible"; DESIGN.md §3 #23):
// the linear map from the s values at the Chebyshev-Lobatto nodes tau_k = (dT/2)(1 - cos(pi k/(s-1)))
// to the Taylor coefficients p^{(q)}(sigma_i), q < nq, of THE degree-(s-1) interpolant p at the uniform
// piece starts sigma_i = i dT/(s-1):  D[(i*nq + q)*s + k].  Host, once per solve, in long double:
// Chebyshev coefficients by the discrete cosine formula, derivatives by the coefficient recurrence
// d_{j-1} = d_{j+1} + 2 j c_j (scaled by 2/dT), values by the three-term recurrence.
static std::vector<double> cheb_taylor_matrix(int s, int nq, double dT) {
  typedef long double ld;
  const int N = s - 1;
  const ld pi = acosl(-1.0L);
  std::vector<double> D(size_t(N) * nq * s, 0.0);
  std::vector<ld> c(N + 1), d(N + 2), Tj(N + 1);
  for (int k = 0; k <= N; ++k) {
    // plain Chebyshev coefficients of the cardinal polynomial of node k: x_k = -cos(pi k/N)
    const ld wk = (k == 0 || k == N) ? 0.5L : 1.0L;
    for (int j = 0; j <= N; ++j) {
      const ld wj = (j == 0 || j == N) ? 0.5L : 1.0L;
      c[j] = wj * (2.0L / N) * wk * cosl(pi * ld(j) * ld(N - k) / ld(N));
    }
    for (int q = 0; q < nq; ++q) {
      if (q > 0) {  // c <- coefficients of dp/dtau
        std::fill(d.begin(), d.end(), 0.0L);
        for (int j = N; j >= 1; --j) d[j - 1] = d[j + 1] + 2.0L * j * c[j];
        d[0] *= 0.5L;
        for (int j = 0; j <= N; ++j) c[j] = d[j] * (2.0L / ld(dT));
      }
      for (int i = 0; i < N; ++i) {
        const ld x = 2.0L * ld(i) / ld(N) - 1.0L;
        Tj[0] = 1.0L;
        if (N >= 1) Tj[1] = x;
        for (int j = 2; j <= N; ++j) Tj[j] = 2.0L * x * Tj[j - 1] - Tj[j - 2];
        ld v = 0.0L;
        for (int j = N; j >= 0; --j) v += c[j] * Tj[j];
        D[(size_t(i) * nq + q) * s + k] = double(v);
      }
    }
  }
  return D;
}

// Two-pass Gram SVD (subsystem 3) of E sample matrices G [E][s][n]; writes V block 0
// (mmax columns, orthonormal), coef, crit into B and returns mmax (host).
static int svd_stage(cudaStream_t st, SvdBufs& S, EbkBufs* B, int E, int n, int s, const double* G, double tau,
                     double eta, double h, int* me_host) {
  const long long gs_e = (long long)s * n;
  const double theta = 1e-6;
  int npass = std::max(1, (int)std::ceil(std::log(0.5 * tau) / std::log(theta)));
  npass = std::min(npass, 4);
  double* part = B->part;
  size_t part_cap = B->part_cap;
  PEXP_CUDA_TRY(cudaMemsetAsync(B->xcnt, 0, E * sizeof(int), st));
  launch_fill_i32(st, S.off, E, 0);
  double* U = S.U;   // current orthonormal basis: columns [0, ko) valid (zero beyond off[e])
  double* Fr = S.R;  // free buffer
  int ko = 0;        // max over evaluations of off[e] (host copy, read back after each selection)
  std::vector<int> offh(E);
  for (int p = 0; p < npass; ++p) {
    const double* X = G;
    if (p > 0 && ko > 0) {
      // residual R = G - U (U^T G), explicit (pass p resolves what pass p-1 could not)
      launch_xty(st, E, n, U, gs_e, 0, ko, G, gs_e, 0, s, part, part_cap, S.Cb, (long long)s * s, ko, 0, 0, false,
                 nullptr, B->xcnt);
      PEXP_CUDA_TRY(cudaMemcpyAsync(Fr, G, size_t(E) * s * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      launch_combine(st, E, n, U, gs_e, 0, ko, S.Cb, (long long)s * s, ko, Fr, gs_e, 0, s, -1.0, 1.0, nullptr);
      X = Fr;
    }
    launch_xty(st, E, n, X, gs_e, 0, s, X, gs_e, 0, s, part, part_cap, S.Gs, (long long)s * s, s, 0, 0, false, nullptr, B->xcnt);
    launch_sym_eig_select(st, E, s, S.Gs, S.lam, S.Msel, S.off, S.sigma1, p, tau, theta, nullptr);
    PEXP_CUDA_TRY(cudaMemcpyAsync(offh.data(), S.off, E * sizeof(int), cudaMemcpyDeviceToHost, st));
    host_sync(st);
    int kn = 0;
    for (int e = 0; e < E; ++e) kn = std::max(kn, offh[e]);
    if (kn == 0) break;  // all-zero samples: nothing selected
    // U[:, 0:ko] += X Msel[:, 0:ko];  U[:, ko:kn] = X Msel[:, ko:kn]
    if (ko > 0) launch_combine(st, E, n, X, gs_e, 0, s, S.Msel, (long long)s * s, s, U, gs_e, 0, ko, 1.0, 1.0, nullptr);
    if (kn > ko)
      launch_combine(st, E, n, X, gs_e, 0, s, S.Msel + size_t(ko) * s, (long long)s * s, s, U, gs_e, ko, kn - ko, 1.0,
                     0.0, nullptr);
    ko = kn;
    // CholQR2 of U[:, 0:ko] (masked: zero columns stay zero); ping-pong U <-> Fr
    for (int q = 0; q < 2; ++q) {
      launch_xty(st, E, n, U, gs_e, 0, ko, U, gs_e, 0, ko, part, part_cap, S.Gs, (long long)ko * ko, ko, 0, 0, false,
                 nullptr, B->xcnt);
      launch_block_chol(st, E, ko, S.Gs, (long long)ko * ko, ko, nullptr, 0, 0, 0.0, S.Rinv, nullptr, 0, 0, nullptr, 0, 0,
                        nullptr, 0, nullptr, false);
      launch_combine(st, E, n, U, gs_e, 0, ko, S.Rinv, (long long)ko * ko, ko, Fr, gs_e, 0, ko, 1.0, 0.0, nullptr);
      std::swap(U, Fr);
    }
  }
  // C = U^T G (rows 0..ko-1 of the s x s matrix Cb), one-sided Jacobi SVD, truncation
  if (ko > 0)
    launch_xty(st, E, n, U, gs_e, 0, ko, G, gs_e, 0, s, part, part_cap, S.Cb, (long long)s * s, s, 0, 0, false, nullptr,
               B->xcnt);
  launch_onesided_svd(st, E, s, S.Cb, S.off, tau, S.Qs, S.sig, S.Cs, S.me, nullptr);
  std::vector<int> mh(E);
  PEXP_CUDA_TRY(cudaMemcpyAsync(mh.data(), S.me, E * sizeof(int), cudaMemcpyDeviceToHost, st));
  host_sync(st);
  int mmax = 0;
  for (int e = 0; e < E; ++e) mmax = std::max(mmax, mh[e]);
  if (me_host) std::copy(mh.begin(), mh.end(), me_host);
  if (!B) return mmax;
  const int mb = std::max(mmax, 1);
  if (mb > B->mcap) fail(1, "retained rank exceeds capacity");
  launch_build_final(st, E, s, mb, S.off, S.Qs, S.sig, S.Cs, S.me, S.Msel, S.Cfin, S.fill);
  // final block U_j (mb columns, padded with the next singular vectors / random columns),
  // CholQR2 -> S.U (stride s*n); the EBK copies each chunk's U_j into its basis block 0
  if (ko > 0)
    launch_combine(st, E, n, U, gs_e, 0, ko, S.Msel, (long long)s * mb, s, Fr, gs_e, 0, mb, 1.0, 0.0, nullptr);
  else
    PEXP_CUDA_TRY(cudaMemsetAsync(Fr, 0, size_t(E) * s * n * sizeof(double), st));
  launch_fill_random(st, E, n, mb, S.fill, Fr, gs_e, 12345u);
  for (int q = 0; q < 2; ++q) {
    double* X = q == 0 ? Fr : S.U;
    launch_xty(st, E, n, X, gs_e, 0, mb, X, gs_e, 0, mb, part, part_cap, S.Gs, (long long)mb * mb, mb, 0, 0,
               false, nullptr, B->xcnt);
    launch_block_chol(st, E, mb, S.Gs, (long long)mb * mb, mb, nullptr, 0, 0, 0.0, S.Rinv, nullptr, 0, 0, nullptr, 0,
                      0, nullptr, 0, nullptr, false);
    if (q == 0) {
      launch_combine(st, E, n, Fr, gs_e, 0, mb, S.Rinv, (long long)mb * mb, mb, S.U, gs_e, 0, mb, 1.0, 0.0, nullptr);
    } else if (mb <= 32) {
      launch_combine(st, E, n, S.U, gs_e, 0, mb, S.Rinv, (long long)mb * mb, mb, S.U, gs_e, 0, mb, 1.0, 0.0, nullptr);
    } else {
      launch_combine(st, E, n, S.U, gs_e, 0, mb, S.Rinv, (long long)mb * mb, mb, Fr, gs_e, 0, mb, 1.0, 0.0, nullptr);
      PEXP_CUDA_TRY(cudaMemcpyAsync(S.U, Fr, size_t(E) * gs_e * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
  }
  if (g_cfg.node_rule == 1) {
    if (!S.pt_ready) h2d(st, S.Dmat, cheb_taylor_matrix(s, g_cfg.nq, h * (s - 1)));
    launch_poly_coef(st, E, s, mb, g_cfg.nq, S.Dmat, S.Cfin, eta, B->coef, B->crit);
  } else {
    if (!S.pt_ready) h2d(st, S.Kinv, notaknot_inverse(s));  // once per solve (depends on s only)
    launch_spline(st, E, s, mb, S.Kinv, S.Cfin, h, eta, B->coef, B->crit);
  }
  S.pt_ready = true;
  k_active_from_m<<<cdiv(E, 256), 256, 0, st>>>(E, S.me, B->active);
  count_launch();
  PEXP_LAUNCH_CHECK();
  return mmax;
}

}  // namespace pexp

using namespace pexp;

// ---------------------------------------------------------------- context
struct pexp_ctx {
  int64_t n = 0;
  int bc = 0;
  int batch = 1;
  std::vector<double> nu, a;
  pexp_options opt{};
  char* ws = nullptr;
  size_t ws_bytes = 0;
  std::string err;
  // side stream + events: the shift-and-invert factorisation runs concurrently with the source
  // SVD stage (they are independent until the block Arnoldi starts)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~pexp_ctx() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
  }
};

// Launch the factorisation on the context's side stream after everything queued on st so far;
// join() makes st wait for it.
struct SideFactor {
  pexp_ctx* c;
  cudaStream_t st;
  SideFactor(pexp_ctx* c_, cudaStream_t st_) : c(c_), st(st_) {
    if (!c->side) {
      PEXP_CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      PEXP_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      PEXP_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    PEXP_CUDA_TRY(cudaEventRecord(c->ev_fork, st));
    PEXP_CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  }
  cudaStream_t stream() const { return c->side; }
  void join() {
    PEXP_CUDA_TRY(cudaEventRecord(c->ev_join, c->side));
    PEXP_CUDA_TRY(cudaStreamWaitEvent(st, c->ev_join, 0));
  }
};

static pexp_status set_err(pexp_ctx* c, int code, const std::string& m) {
  if (c) c->err = m;
  return (pexp_status)code;
}

template <class F>
static pexp_status guarded(pexp_ctx* c, F&& f) {
  try {
    f();
    if (c) c->err.clear();
    return PEXP_OK;
  } catch (const Error& e) {
    return set_err(c, e.code, e.msg);
  } catch (const std::exception& e) {
    return set_err(c, PEXP_EINVAL, e.what());
  }
}

// Homogeneous legs per group (one shared block Krylov space per group; <= 16, KSMALL limits).
// pexp_options.hom_group, default 8 (measured on C2: 8 legs per group beat 16, 48 vs 58 ms).
static int hom_group_width(const pexp_ctx* c, int P) {
  const int w = c->opt.hom_group > 0 ? std::min(c->opt.hom_group, 16) : 8;
  return std::max(1, std::min(w, P - 1));
}

// Two CUDA events of a timed call, destroyed on every exit path (errors throw).
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  EventPair() {
    PEXP_CUDA_TRY(cudaEventCreate(&a));
    PEXP_CUDA_TRY(cudaEventCreate(&b));
  }
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  float ms() {
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    return t;
  }
};

// ---------------------------------------------------------------- workspace plans
struct LinPlan {
  Ops O;
  Factors F;
  double *nu_d, *a_d, *gam_f, *Au0, *G, *Yend, *Yh;
  int *opidx_f, *err, *iota;
  SvdBufs S;
  EbkBufs B, Bh;
};

static void plan_linear(Arena& ar, LinPlan& L, const pexp_ctx* c, int P) {
  Opts o = norm_opts(c->opt);
  const int n = (int)c->n, Bt = c->batch, s = o.s, E = Bt * P, Eh = Bt * (P - 1);
  L.O.n = n; L.O.nops = Bt;
  L.O.sub = ar.take<double>(size_t(Bt) * n);
  L.O.diag = ar.take<double>(size_t(Bt) * n);
  L.O.sup = ar.take<double>(size_t(Bt) * n);
  L.F.n = n; L.F.nf = 2 * Bt; L.F.periodic = c->bc == PEXP_BC_PERIODIC;
  L.F.l = ar.take<double>(size_t(2 * Bt) * n);
  L.F.dinv = ar.take<double>(size_t(2 * Bt) * n);
  L.F.sup = ar.take<double>(size_t(2 * Bt) * n);
  L.F.z = ar.take<double>(size_t(2 * Bt) * n);
  L.F.w = ar.take<double>(size_t(2 * Bt) * n);
  L.nu_d = ar.take<double>(Bt);
  L.a_d = ar.take<double>(Bt);
  L.gam_f = ar.take<double>(2 * Bt);
  L.opidx_f = ar.take<int>(2 * Bt);
  L.err = ar.take<int>(4);
  L.iota = ar.take<int>(std::max(Bt, 1));
  L.Au0 = ar.take<double>(size_t(Bt) * n);
  L.G = ar.take<double>(size_t(E) * s * n);
  L.Yend = ar.take<double>(size_t(E) * n);
  alloc_svd(ar, L.S, E, n, s);
  const bool restartable = o.restart_blocks > 0 || o.kcyc < o.kcap;
  alloc_ebk(ar, L.B, E, o.chunk, n, o.kcyc, o.kcap, s, 2, s, true, L.S.R, restartable, 1, o.nq);
  if (P > 1) {
    const int mh = hom_group_width(c, P), G = cdiv(P - 1, mh), Eg = Bt * G;
    // a group of mh legs needs a wider space than one forced evaluation (measured on C2:
    // 16 legs -> 288 columns); give it at least 24 block steps
    const int kcap_h = std::min(KSMALL_MAX - 64, std::max(o.kcap, 24 * mh));
    alloc_ebk(ar, L.Bh, Eg, Eg, n, kcap_h, kcap_h, mh, P, s, false, nullptr, false);
    L.Bh.groups = G;
    L.Yh = ar.take<double>(size_t(Eg) * P * n);
  } else {
    L.Yh = nullptr;
  }
  (void)Eh;
}

struct BurPlan {
  Ops O;
  Factors F, Fs;            // Fs: factorisations with the scan's own shift (scan_gamma_factor != 1)
  double* gam_s = nullptr;  // [P] scan shifts
  double *Uk, *Un, *ubar, *G, *Y, *Wh, *uhat, *delta;
  int *iota, *err;
  char* scan_ws = nullptr;
  size_t scan_bytes = 0;
  SvdBufs S;
  EbkBufs B, B1;
};

static void plan_burgers(Arena& ar, BurPlan& L, const pexp_ctx* c, int P) {
  Opts o = norm_opts(c->opt);
  const int n = (int)c->n, s = o.s, E = P;
  L.O.n = n; L.O.nops = P;
  L.O.sub = ar.take<double>(size_t(P) * n);
  L.O.diag = ar.take<double>(size_t(P) * n);
  L.O.sup = ar.take<double>(size_t(P) * n);
  L.F.n = n; L.F.nf = P; L.F.periodic = 1;
  L.F.l = ar.take<double>(size_t(P) * n);
  L.F.dinv = ar.take<double>(size_t(P) * n);
  L.F.sup = ar.take<double>(size_t(P) * n);
  L.F.z = ar.take<double>(size_t(P) * n);
  L.F.w = ar.take<double>(size_t(P) * n);
  if (c->opt.scan_gamma_factor > 0 && c->opt.scan_gamma_factor != 1.0) {  // the scan's own shift
    L.Fs = L.F;
    L.Fs.l = ar.take<double>(size_t(P) * n);
    L.Fs.dinv = ar.take<double>(size_t(P) * n);
    L.Fs.sup = ar.take<double>(size_t(P) * n);
    L.Fs.z = ar.take<double>(size_t(P) * n);
    L.Fs.w = ar.take<double>(size_t(P) * n);
    L.gam_s = ar.take<double>(P);
  }
  L.Uk = ar.take<double>(size_t(P) * s * n);
  L.Un = ar.take<double>(size_t(P) * s * n);
  L.ubar = ar.take<double>(size_t(P) * n);
  L.G = ar.take<double>(size_t(P) * s * n);
  L.Y = ar.take<double>(size_t(P) * s * n);
  L.Wh = ar.take<double>(size_t(s) * n);
  L.uhat = ar.take<double>(n);
  L.delta = ar.take<double>(4);
  L.iota = ar.take<int>(P);
  L.err = ar.take<int>(4);
  alloc_svd(ar, L.S, E, n, s);
  const bool restartable = o.restart_blocks > 0 || o.kcyc < o.kcap;
  alloc_ebk(ar, L.B, E, o.chunk, n, o.kcyc, o.kcap, s, s, s, true, L.S.R, restartable, s);
  const int k1 = std::min(o.kcap, 512);  // scan: single vectors, short spaces, no restart
  alloc_ebk(ar, L.B1, 1, 1, n, k1, k1, 1, s, s, false, nullptr, false);
  if (hom_scan_ok(n, k1)) {
    L.scan_bytes = hom_scan_bytes(n, s, k1, P);
    L.scan_ws = ar.take<char>(L.scan_bytes);
  }
}

static size_t lin_bytes(const pexp_ctx* c, int P) {
  Arena ar;
  LinPlan L;
  plan_linear(ar, L, c, P);
  return ar.off;
}
static size_t bur_bytes(const pexp_ctx* c, int P) {
  if (c->bc != PEXP_BC_PERIODIC || c->batch != 1) return 0;
  Arena ar;
  BurPlan L;
  plan_burgers(ar, L, c, P);
  return ar.off;
}

// One-time per-device kernel attributes (> 48 KB dynamic shared memory, cluster sizes).
static void init_once() {
  static unsigned long long done = 0;  // bit d: device d initialised
  int dev = 0;
  PEXP_CUDA_TRY(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(done & bit)) {
    tsmm_init();
    small_init();
    stream_init();
    done |= bit;
  }
}

// Smallest Krylov dimension the evaluations idx[0..cnt) (or first..first+cnt) needed in the previous WR
// iteration (g_cfg.kprev), 0 if unknown.
static int kprev_min(const int* idx, int first, int cnt) {
  if (!g_cfg.kprev) return 0;
  int mn = 1 << 30;
  for (int i = 0; i < cnt; ++i) {
    const int k = g_cfg.kprev[idx ? idx[i] : first + i];
    if (k > 0) mn = std::min(mn, k);
  }
  return mn == (1 << 30) ? 0 : mn;
}

// The forced EBK over E evaluations in chunks of B.E (eval_chunk): each chunk copies its
// U_j from the SVD stage into basis block 0, runs the block Arnoldi, and writes its outputs
// Y[e] (+)= V_e z_e at output o0 (restart accumulation, then the final cycle).
static RunInfo ebk_forced_chunked(cudaStream_t st, EbkBufs& B, const SvdBufs& S, const Factors& F, const Ops& O,
                                  bool periodic, int E, int mmax, double h, int s, int out_stride, int nout,
                                  int o0, double* Y, long long ys_e, int stop_rule, int restart_blocks) {
  RunInfo tot;
  const int n = B.n, Ecap = B.E;
  const int no = o0 == 0 ? nout : 1;
  for (int c0 = 0; c0 < E; c0 += Ecap) {
    const int ec = std::min(Ecap, E - c0);
    EbkBufs Bc = chunk_view(B, c0, ec, mmax);
    PEXP_CUDA_TRY(cudaMemcpy2DAsync(Bc.V, Bc.vs_e * sizeof(double), S.U + size_t(c0) * s * n,
                                    size_t(s) * n * sizeof(double), size_t(mmax) * n * sizeof(double), ec,
                                    cudaMemcpyDeviceToDevice, st));
    double* Yc = Y + size_t(c0) * ys_e;
    RunInfo r = ebk_run(st, Bc, F, O, periodic, mmax, 0, h, s - 1, out_stride, nout, stop_rule,
                        Accum{Yc, ys_e, o0, no}, restart_blocks, kprev_min(nullptr, c0, ec));
    launch_combine(st, ec, n, Bc.V, Bc.vs_e, 0, std::max(r.max_k, 1), Bc.Z + size_t(o0) * Bc.kcap, Bc.zs_e, Bc.kcap,
                   Yc, ys_e, 0, no, 1.0, r.restarts ? 1.0 : 0.0, nullptr, Bc.kfin);
    tot.max_k = std::max(tot.max_k, r.max_k);
    tot.max_ktot = std::max(tot.max_ktot, r.max_ktot);
    tot.restarts += r.restarts;
    tot.unconverged += r.unconverged;
    tot.worst_res_ratio = std::max(tot.worst_res_ratio, r.worst_res_ratio);
  }
  return tot;
}

// Width buckets: evaluations are grouped by their retained rank m_j rounded up
// to a multiple of 4, and every bucket runs its own block Arnoldi with that block width instead of
// padding every evaluation to max_j m_j (the Krylov dimension, bytes and flops grow with the block
// width).  Buckets with fewer than 16 evaluations merge into the next wider one.  Each chunk
// gathers its evaluations' inputs into chunk slots, runs the EBK, and scatters the outputs (and the
// k_j records) back.  The projected solution of an evaluation does not depend on its padding
// (padding columns carry zero coefficients), only the Krylov space it is found in.
static std::vector<std::pair<int, std::vector<int>>> width_buckets(const int* me, int E, int mmax) {
  std::vector<std::vector<int>> cls((mmax + 3) / 4 + 1);
  for (int e = 0; e < E; ++e) cls[me[e] <= 0 ? 0 : (me[e] + 3) / 4].push_back(e);
  // zero-rank evaluations (inactive) ride with the narrowest non-empty class
  std::vector<std::pair<int, std::vector<int>>> out;
  std::vector<int> carry = cls[0];
  for (size_t c = 1; c < cls.size(); ++c) {
    carry.insert(carry.end(), cls[c].begin(), cls[c].end());
    const bool last = c + 1 == cls.size();
    if (carry.empty()) continue;
    int ncarry_active = 0;
    for (int e : carry) ncarry_active += me[e] > 0;
    if (ncarry_active >= 16 || last) {
      out.push_back({std::min(int(4 * c), mmax), carry});
      carry.clear();
    }
  }
  if (!carry.empty()) {
    if (out.empty()) out.push_back({std::max(mmax, 1), carry});
    else out.back().second.insert(out.back().second.end(), carry.begin(), carry.end());
  }
  return out;
}

static RunInfo ebk_forced_bucketed(cudaStream_t st, EbkBufs& B, const SvdBufs& S, const Factors& F, const Ops& O,
                                   bool periodic, int E, int mmax, const int* me, double h, int s, int out_stride,
                                   int nout, int o0, double* Y, long long ys_e, int stop_rule, int restart_blocks) {
  RunInfo tot;
  const int n = B.n, Ecap = B.E;
  const int no = o0 == 0 ? nout : 1;
  if (no > B.ycols) fail(1, "bucketed EBK: output staging too small");
  auto buckets = width_buckets(me, E, mmax);
  std::vector<int> perm;
  for (auto& b : buckets) perm.insert(perm.end(), b.second.begin(), b.second.end());
  PEXP_CUDA_TRY(cudaMemcpyAsync(B.perm, perm.data(), E * sizeof(int), cudaMemcpyHostToDevice, st));
  host_sync(st);  // pageable source
  int p0 = 0;
  for (auto& bk : buckets) {
    const int wb = bk.first, nb = int(bk.second.size());
    for (int c0 = 0; c0 < nb; c0 += Ecap) {
      const int ec = std::min(Ecap, nb - c0);
      GatherArgs ga{};
      ga.perm = B.perm + p0; ga.wb = wb; ga.mmax = std::max(mmax, 1); ga.s = s; ga.n = n; ga.nq = B.nq;
      ga.gam = B.gam; ga.crit = B.crit; ga.coef = B.coef; ga.U = S.U; ga.us_e = (long long)s * n;
      ga.active = B.active; ga.fidx = B.fidx; ga.opidx = B.opidx;
      ga.gam_c = B.gam_c; ga.crit_c = B.crit_c; ga.coef_c = B.coef_c; ga.V = B.V; ga.vs_e = B.vs_e;
      ga.active_c = B.active_c; ga.fidx_c = B.fidx_c; ga.opidx_c = B.opidx_c;
      launch_bucket_gather(st, ec, ga);
      EbkBufs Bc = B;
      Bc.E = ec;
      Bc.gam = B.gam_c; Bc.crit = B.crit_c; Bc.coef = B.coef_c; Bc.active = B.active_c;
      Bc.fidx = B.fidx_c; Bc.opidx = B.opidx_c; Bc.krec = B.krec_c;
      launch_fill_i32(st, Bc.krec, ec, 0);
      const long long yts = (long long)no * n;
      // restart cycles keep the column count of the unbucketed run: restart_blocks steps of max m_j
      const int rb = restart_blocks > 0 ? cdiv(long(restart_blocks) * std::max(mmax, 1), wb) : restart_blocks;
      RunInfo r = ebk_run(st, Bc, F, O, periodic, wb, 0, h, s - 1, out_stride, nout, stop_rule,
                          Accum{B.Ytmp, yts, o0, no}, rb, kprev_min(perm.data() + p0, 0, ec));
      launch_combine(st, ec, n, Bc.V, Bc.vs_e, 0, std::max(r.max_k, 1), Bc.Z + size_t(o0) * Bc.kcap, Bc.zs_e, Bc.kcap,
                     B.Ytmp, yts, 0, no, 1.0, r.restarts ? 1.0 : 0.0, nullptr, Bc.kfin);
      launch_bucket_scatter(st, ec, B.perm + p0, size_t(no) * n, B.Ytmp, yts, Y, ys_e, B.krec_c, B.krec);
      tot.max_k = std::max(tot.max_k, r.max_k);
      tot.max_ktot = std::max(tot.max_ktot, r.max_ktot);
      tot.restarts += r.restarts;
      tot.unconverged += r.unconverged;
      tot.worst_res_ratio = std::max(tot.worst_res_ratio, r.worst_res_ratio);
      ++tot.chunks;
      p0 += ec;
    }
  }
  tot.buckets = int(buckets.size());
  return tot;
}

// The forced EBK: width buckets when the retained ranks differ enough to pay for them.
static RunInfo ebk_forced(cudaStream_t st, EbkBufs& B, const SvdBufs& S, const Factors& F, const Ops& O, bool periodic,
                          int E, int mmax, const int* me, double h, int s, int out_stride, int nout, int o0, double* Y,
                          long long ys_e, int stop_rule, int restart_blocks) {
  if (B.perm && g_cfg.buckets && width_buckets(me, E, mmax).size() > 1)
    return ebk_forced_bucketed(st, B, S, F, O, periodic, E, mmax, me, h, s, out_stride, nout, o0, Y, ys_e, stop_rule,
                               restart_blocks);
  return ebk_forced_chunked(st, B, S, F, O, periodic, E, mmax, h, s, out_stride, nout, o0, Y, ys_e, stop_rule,
                            restart_blocks);
}

// ---------------------------------------------------------------- C ABI
extern "C" {

pexp_status pexp_create(pexp_ctx** ctx, int64_t n, pexp_bc bc, double nu, double a, const pexp_options* opt) {
  return pexp_create_batched(ctx, n, bc, 1, &nu, &a, opt);
}

pexp_status pexp_create_batched(pexp_ctx** ctx, int64_t n, pexp_bc bc, int32_t batch, const double* nu_host,
                                const double* a_host, const pexp_options* opt) {
  if (!ctx) return PEXP_EINVAL;
  *ctx = nullptr;
  if (n < 3 || n > (1LL << 30)) return PEXP_EINVAL;
  if (bc != PEXP_BC_PERIODIC && bc != PEXP_BC_DIRICHLET) return PEXP_EINVAL;
  if (batch < 1 || !nu_host || !a_host) return PEXP_EINVAL;
  for (int b = 0; b < batch; ++b)
    if (!(nu_host[b] >= 0.0) || !std::isfinite(nu_host[b]) || !std::isfinite(a_host[b])) return PEXP_EINVAL;
  pexp_options o{};
  if (opt) o = *opt;
  if (o.s != 0 && (o.s < 4 || o.s > 64)) return PEXP_EINVAL;
  if (o.node_rule < 0 || o.node_rule > 1) return PEXP_EINVAL;
  if (o.k_max < 0 || o.k_max > KSMALL_MAX - 64) return PEXP_EINVAL;
  // projected-problem capacity: K + nq*m <= KSMALL_MAX with m <= s (node_rule 1: nq = 12)
  if (o.node_rule == 1 && (o.k_max > 0 ? o.k_max : 256) + NQ_CHEB * (o.s > 0 ? o.s : 32) > KSMALL_MAX) return PEXP_EINVAL;
  if (o.stop_rule < 0 || o.stop_rule > 1) return PEXP_EINVAL;
  if (o.basis_cols < 0 || o.eval_chunk < 0) return PEXP_EINVAL;
  if (o.route < 0 || o.route > 2 || o.defl_tol < 0 || o.piv_tol < 0 || o.hom_group < 0 || o.hom_group > 16)
    return PEXP_EINVAL;
  if (o.width_buckets < -1 || o.width_buckets > 1) return PEXP_EINVAL;
  if (!(o.scan_gamma_factor >= 0.0) || o.scan_gamma_factor > 16.0) return PEXP_EINVAL;
  if (!(o.gamma_factor >= 0.0) || o.gamma_factor > 16.0) return PEXP_EINVAL;
  pexp_ctx* c = new pexp_ctx;
  c->n = n;
  c->bc = bc;
  c->batch = batch;
  c->nu.assign(nu_host, nu_host + batch);
  c->a.assign(a_host, a_host + batch);
  c->opt = o;
  *ctx = c;
  return PEXP_OK;
}

void pexp_destroy(pexp_ctx* ctx) { delete ctx; }

const char* pexp_last_error(const pexp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

pexp_status pexp_sample_times(const pexp_ctx* ctx, double T, int32_t P, double* t_host) {
  if (!ctx || !t_host || !(T > 0) || P < 1) return PEXP_EINVAL;
  Opts o = norm_opts(ctx->opt);
  const double dT = T / P;
  const double pi = std::acos(-1.0);
  for (int j = 0; j < P; ++j)
    for (int i = 0; i < o.s; ++i)
      t_host[size_t(j) * o.s + i] = o.node_rule == 1 ? j * dT + 0.5 * dT * (1.0 - std::cos(pi * i / (o.s - 1)))
                                                     : j * dT + i * (dT / (o.s - 1));
  return PEXP_OK;
}

int32_t pexp_chebyshev_taylor_matrix(const pexp_ctx* ctx, double dT, double* D_host) {
  if (!ctx || !D_host || !(dT > 0) || ctx->opt.node_rule != 1) return 0;
  Opts o = norm_opts(ctx->opt);
  const std::vector<double> D = cheb_taylor_matrix(o.s, o.nq, dT);
  std::copy(D.begin(), D.end(), D_host);
  return o.nq;
}

size_t pexp_workspace_bytes(const pexp_ctx* ctx, int32_t P, int32_t kind) {
  if (!ctx || P < 1 || kind < 0 || kind > 2) return 0;
  if (kind == 0) return lin_bytes(ctx, P) + 256;
  if (kind == 1) return bur_bytes(ctx, P) + 256;
  return std::max(lin_bytes(ctx, P), bur_bytes(ctx, P)) + 256;
}

pexp_status pexp_set_workspace(pexp_ctx* ctx, void* dev_ptr, size_t bytes) {
  if (!ctx) return PEXP_EINVAL;
  if (dev_ptr && (reinterpret_cast<uintptr_t>(dev_ptr) & 255)) return set_err(ctx, PEXP_EINVAL, "workspace must be 256-byte aligned");
  ctx->ws = (char*)dev_ptr;
  ctx->ws_bytes = bytes;
  return PEXP_OK;
}

pexp_status pexp_solve_linear(pexp_ctx* ctx, const double* u0, const double* src, double T, int32_t P, double tol,
                              double* out, pexp_stats* st_out) {
  return pexp_solve_linear_stages(ctx, u0, src, nullptr, T, P, tol, out, nullptr, nullptr, st_out);
}

pexp_status pexp_solve_linear_stages(pexp_ctx* ctx, const double* u0, const double* src, const double* vstart,
                                     double T, int32_t P, double tol, double* out, double* vend, double* legs,
                                     pexp_stats* st_out) {
  if (!ctx) return PEXP_EINVAL;
  if (!u0 || (!src && !vstart) || !out) return set_err(ctx, PEXP_EINVAL, "null array argument");
  if (!(T > 0) || !std::isfinite(T)) return set_err(ctx, PEXP_EINVAL, "T must be > 0");
  if (P < 1) return set_err(ctx, PEXP_EINVAL, "P must be >= 1");
  if (!(tol >= 1e-14 && tol <= 1e-2)) return set_err(ctx, PEXP_EINVAL, "tol must be in [1e-14, 1e-2]");
  if (!ctx->ws) return set_err(ctx, PEXP_ENOMEM, "workspace not set (pexp_set_workspace)");
  if (ctx->ws_bytes < lin_bytes(ctx, P)) return set_err(ctx, PEXP_ENOMEM, "workspace too small for this P");
  return guarded(ctx, [&] {
    init_once();
    g_launches = 0;
    Opts o = norm_opts(ctx->opt);
    g_cfg = o.cfg;
    cudaStream_t st = o.st;
    const int n = (int)ctx->n, Bt = ctx->batch, s = o.s, E = Bt * P, Eh = Bt * (P - 1);
    const bool periodic = ctx->bc == PEXP_BC_PERIODIC;
    const double dT = T / P, h = dT / (s - 1), tau = o.tau_f * tol, eta = o.eta_f * tol;
    Arena ar{ctx->ws, ctx->ws_bytes, 0};
    LinPlan L;
    plan_linear(ar, L, ctx, P);
    EventPair ev;
    PEXP_CUDA_TRY(cudaEventRecord(ev.a, st));
    // operators and factorisations: f < Bt: gamma = dT/10 (nonhomogeneous); f >= Bt: gamma = T/10 (legs)
    h2d(st, L.nu_d, ctx->nu);
    h2d(st, L.a_d, ctx->a);
    launch_ade_rows(st, Bt, n, !periodic, L.nu_d, L.a_d, L.O.sub, L.O.diag, L.O.sup);
    std::vector<double> gf(2 * Bt);
    std::vector<int> of(2 * Bt), iota(Bt);
    const double gfac = ctx->opt.gamma_factor > 0 ? ctx->opt.gamma_factor : 1.0;
    for (int b = 0; b < Bt; ++b) { gf[b] = gfac * dT / 10; gf[Bt + b] = T / 10; of[b] = b; of[Bt + b] = b; iota[b] = b; }
    h2d(st, L.gam_f, gf);
    h2d(st, L.opidx_f, of);
    h2d(st, L.iota, iota);
    PEXP_CUDA_TRY(cudaMemsetAsync(L.err, 0, sizeof(int), st));
    SideFactor sf(ctx, st);
    launch_factor(sf.stream(), L.F, 2 * Bt, L.opidx_f, L.gam_f, L.O, L.err);
    std::vector<int> me(E, 0);
    int mmax = 0;
    if (!vstart) {
      // shifted source G = A u0 + g at the nodes
      launch_apply_A(st, L.O, L.iota, Bt, 1, u0, n, 0, L.Au0, n, 0, periodic);
      launch_lin_source(st, Bt, P, s, n, L.Au0, src, L.G);
      // per-eval maps for the nonhomogeneous batch
      std::vector<int> fe(E);
      std::vector<double> ge(E, gfac * dT / 10);
      for (int e = 0; e < E; ++e) fe[e] = e / P;
      h2d(st, L.B.fidx, fe);
      h2d(st, L.B.opidx, fe);
      h2d(st, L.B.gam, ge);
      mmax = svd_stage(st, L.S, &L.B, E, n, s, L.G, tau, eta, h, me.data());
    }
    sf.join();
    int herr = 0;
    PEXP_CUDA_TRY(cudaMemcpyAsync(&herr, L.err, sizeof(int), cudaMemcpyDeviceToHost, st));
    host_sync(st);
    if (herr) fail(PEXP_EPIVOT, "shift-and-invert factorisation: a pivot is zero relative to its row or non-finite");
    launch_fill_i32(st, L.B.krec, E, 0);
    RunInfo ri{}, rh{};
    if (vstart) {  // stage entry: the homogeneous legs start from the caller's v_j(T_j)
      PEXP_CUDA_TRY(cudaMemcpyAsync(L.Yend, vstart, size_t(E) * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    } else if (mmax > 0) {
      ri = ebk_forced(st, L.B, L.S, L.F, L.O, periodic, E, mmax, me.data(), h, s, s - 1, 2, 1, L.Yend, n, o.stop_rule,
                      o.restart_blocks);
    } else {
      PEXP_CUDA_TRY(cudaMemsetAsync(L.Yend, 0, size_t(E) * n * sizeof(double), st));
    }
    if (vend) PEXP_CUDA_TRY(cudaMemcpyAsync(vend, L.Yend, size_t(E) * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    EventPair evh;  // homogeneous legs + superposition (tau_2)
    PEXP_CUDA_TRY(cudaEventRecord(evh.a, st));
    int G = 0;
    if (P > 1) {
      // homogeneous legs, grouped: up to 16 consecutive legs share one block Krylov space
      // (EBK for the homogeneous part too); group eh = b*G + g holds legs
      // j = g*mh .. g*mh+mh-1 of problem b
      const int mh = hom_group_width(ctx, P);
      G = cdiv(P - 1, mh);
      const int Eg = Bt * G;
      EbkBufs& Bh = L.Bh;
      std::vector<int> fh(Eg), oh(Eg);
      std::vector<double> gh(Eg, T / 10);
      for (int e = 0; e < Eg; ++e) { fh[e] = Bt + e / G; oh[e] = e / G; }
      h2d(st, Bh.fidx, fh);
      h2d(st, Bh.opidx, oh);
      h2d(st, Bh.gam, gh);
      launch_hom_start_block(st, Eg, mh, G, P, n, L.Yend, Bh.V, Bh.vs_e, Bh.beta);
      // block 0 = orthonormal basis Q of the start vectors Y0 (robust pivoted/deferred in-block
      // QR, legs below 1e-10 of their own norm deflated), z0 = R0 = Q^T Y0 (exact to eps)
      PEXP_CUDA_TRY(cudaMemsetAsync(Bh.xcnt, 0, Eg * sizeof(int), st));
      PEXP_CUDA_TRY(cudaMemcpy2DAsync(Bh.Wt, size_t(mh) * n * sizeof(double), Bh.V, Bh.vs_e * sizeof(double),
                                      size_t(mh) * n * sizeof(double), Eg, cudaMemcpyDeviceToDevice, st));
      launch_xty(st, Eg, n, Bh.V, Bh.vs_e, 0, mh, Bh.V, Bh.vs_e, 0, mh, Bh.part, Bh.part_cap, Bh.G0,
                 (long long)mh * mh, mh, 0, 0, false, nullptr, Bh.xcnt);
      const double defl_h = g_cfg.defl;
      inblock_qr(st, Bh, Eg, n, mh, 0, Bh.G0, (long long)mh * mh, mh, defl_h, nullptr);
      chol_combine_block(st, Bh, Eg, n, mh, 0, nullptr, 0, 0, 0.0, defl_h, nullptr, nullptr);
      launch_xty(st, Eg, n, Bh.V, Bh.vs_e, 0, mh, Bh.Wt, (long long)mh * n, 0, mh, Bh.part, Bh.part_cap, Bh.R0,
                 (long long)mh * mh, mh, 0, 0, false, nullptr, Bh.xcnt);
      launch_hom_setup_block(st, Eg, mh, G, P, dT, eta, Bh.beta, Bh.critc, Bh.horc, Bh.active);
      rh = ebk_run(st, Bh, L.F, L.O, periodic, mh, 2, dT, 0, 1, P, o.stop_rule);
      launch_combine(st, Eg, n, Bh.V, Bh.vs_e, 0, std::max(rh.max_k, 1), Bh.Z, Bh.zs_e, Bh.kcap, L.Yh,
                     (long long)P * n, 0, P, 1.0, 0.0, nullptr, Bh.kfin);
    }
    if (legs && P > 1)
      PEXP_CUDA_TRY(cudaMemcpyAsync(legs, L.Yh, size_t(Bt) * G * P * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    launch_superpose(st, Bt, P, n, u0, L.Yend, P > 1 ? L.Yh : nullptr, (long long)P * n, n, G, out);
    PEXP_CUDA_TRY(cudaEventRecord(evh.b, st));
    PEXP_CUDA_TRY(cudaEventRecord(ev.b, st));
    PEXP_CUDA_TRY(cudaEventSynchronize(ev.b));
    ++g_cfg.syncs;
    const float ms = ev.ms();
    check_err(st);
    if (st_out) {
      int32_t *mj = st_out->m_j, *kj = st_out->k_j, *ksj = st_out->kscan_j;
      double* gj = st_out->gamma_j;
      std::memset(st_out, 0, sizeof(*st_out));
      st_out->m_j = mj; st_out->k_j = kj; st_out->gamma_j = gj; st_out->kscan_j = ksj;
      if (mj) std::copy(me.begin(), me.end(), mj);
      if (kj) {
        PEXP_CUDA_TRY(cudaMemcpy(kj, L.B.krec, E * sizeof(int), cudaMemcpyDeviceToHost));
        ++g_cfg.syncs;
      }
      if (gj) std::fill(gj, gj + E, gfac * dT / 10);
      st_out->max_m = mmax;
      st_out->max_k = std::max(ri.max_ktot, rh.max_ktot);
      st_out->restarts = ri.restarts;
      st_out->best_residual = std::max(ri.worst_res_ratio, rh.worst_res_ratio);
      st_out->ms_total = ms;
      st_out->ms_hom = evh.ms();
      st_out->ms_nonhom = ms - st_out->ms_hom;
      st_out->evals = E;
      st_out->kernel_launches = (int)g_launches;
      st_out->host_syncs = g_cfg.syncs;
    }
    if (ri.unconverged || rh.unconverged)
      fail(PEXP_ENOCONV, "Krylov capacity k_max reached before the residual target (" +
                             std::to_string(ri.unconverged) + " nonhomogeneous, " + std::to_string(rh.unconverged) +
                             " homogeneous evaluations; worst residual/target " +
                             std::to_string(std::max(ri.worst_res_ratio, rh.worst_res_ratio)) + ", max_k " +
                             std::to_string(std::max(ri.max_ktot, rh.max_ktot)) + ", m " + std::to_string(mmax) + ")");
  });
}

pexp_status pexp_solve_burgers(pexp_ctx* ctx, const double* u0, double nu, double T, int32_t P, double tol,
                               int32_t max_wr_iters, double* out, pexp_stats* st_out) {
  return pexp_solve_burgers_forced(ctx, u0, nullptr, nu, T, P, tol, max_wr_iters, out, st_out);
}

static pexp_status burgers_impl(pexp_ctx* ctx, const double* u0, const double* f, const double* Uinit, double nu,
                                double T, int32_t P, double tol, int32_t max_wr_iters, double* out, double* Uout,
                                pexp_stats* st_out);

pexp_status pexp_solve_burgers_forced(pexp_ctx* ctx, const double* u0, const double* f, double nu, double T,
                                      int32_t P, double tol, int32_t max_wr_iters, double* out,
                                      pexp_stats* st_out) {
  return burgers_impl(ctx, u0, f, nullptr, nu, T, P, tol, max_wr_iters, out, nullptr, st_out);
}

pexp_status pexp_wr_map(pexp_ctx* ctx, const double* u0, const double* f, const double* Uk, double nu, double T,
                        int32_t P, double tol, double* Unew, double* out, pexp_stats* st_out) {
  if (!Uk || !Unew) return set_err(ctx, PEXP_EINVAL, "null array argument");
  return burgers_impl(ctx, u0, f, Uk, nu, T, P, tol, 1, out, Unew, st_out);
}

static pexp_status burgers_impl(pexp_ctx* ctx, const double* u0, const double* f, const double* Uinit, double nu,
                                double T, int32_t P, double tol, int32_t max_wr_iters, double* out, double* Uout,
                                pexp_stats* st_out) {
  if (!ctx) return PEXP_EINVAL;
  if (!u0 || !out) return set_err(ctx, PEXP_EINVAL, "null array argument");
  if (ctx->bc != PEXP_BC_PERIODIC || ctx->batch != 1)
    return set_err(ctx, PEXP_EINVAL, "Burgers requires a periodic context with batch 1");
  if (ctx->opt.node_rule != 0)
    return set_err(ctx, PEXP_EINVAL, "Burgers requires uniform sample nodes (node_rule 0)");
  if (!(nu > 0) || !std::isfinite(nu)) return set_err(ctx, PEXP_EINVAL, "nu must be > 0");
  if (!(T > 0)) return set_err(ctx, PEXP_EINVAL, "T must be > 0");
  if (P < 1) return set_err(ctx, PEXP_EINVAL, "P must be >= 1");
  if (!(tol >= 1e-14 && tol <= 1e-2)) return set_err(ctx, PEXP_EINVAL, "tol must be in [1e-14, 1e-2]");
  if (max_wr_iters < 1) return set_err(ctx, PEXP_EINVAL, "max_wr_iters must be >= 1");
  if (!ctx->ws) return set_err(ctx, PEXP_ENOMEM, "workspace not set (pexp_set_workspace)");
  if (ctx->ws_bytes < bur_bytes(ctx, P)) return set_err(ctx, PEXP_ENOMEM, "workspace too small for this P");
  return guarded(ctx, [&] {
    init_once();
    g_launches = 0;
    Opts o = norm_opts(ctx->opt);
    g_cfg = o.cfg;
    cudaStream_t st = o.st;
    const int n = (int)ctx->n, s = o.s, E = P;
    const double dT = T / P, h = dT / (s - 1), tau = o.tau_f * tol, eta = o.eta_f * tol;
    const double wr_tol = 1e-6;
    const double gfac = ctx->opt.gamma_factor > 0 ? ctx->opt.gamma_factor : 1.0;
    Arena ar{ctx->ws, ctx->ws_bytes, 0};
    BurPlan L;
    plan_burgers(ar, L, ctx, P);
    EventPair ev;
    PEXP_CUDA_TRY(cudaEventRecord(ev.a, st));
    int32_t* rec_m = st_out ? st_out->m_j : nullptr;
    int32_t* rec_k = st_out ? st_out->k_j : nullptr;
    double* rec_g = st_out ? st_out->gamma_j : nullptr;
    int32_t* rec_ks = st_out ? st_out->kscan_j : nullptr;
    std::vector<double> dhist;
    double scan_diag[3] = {0.0, 0.0, 0.0};
    std::vector<int> kprev(P, 0), kcur(P, 0);
    std::vector<std::unique_ptr<EventPair>> scan_ev;  // homogeneous scan + waveform update per iteration
    std::vector<int> iota(P);
    for (int j = 0; j < P; ++j) iota[j] = j;
    h2d(st, L.iota, iota);
    h2d(st, L.B.fidx, iota);
    h2d(st, L.B.opidx, iota);
    if (Uinit)  // stage entry pexp_wr_map: start from the caller's waveform u_k
      PEXP_CUDA_TRY(cudaMemcpyAsync(L.Uk, Uinit, size_t(P) * s * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    else
      launch_broadcast_waveform(st, P, s, n, u0, L.Uk);
    int iters = 0, max_m = 0, max_k = 0, restarts = 0;
    double delta = 0.0, delta0 = -1.0;
    for (int k = 0; k < max_wr_iters; ++k) {
      launch_ubar_gamma(st, P, s, n, L.Uk, gfac * dT / 10, L.ubar, L.B.gam);
      launch_burgers_rows(st, P, n, nu, L.ubar, L.O.sub, L.O.diag, L.O.sup);
      PEXP_CUDA_TRY(cudaMemsetAsync(L.err, 0, sizeof(int), st));
      SideFactor sf(ctx, st);
      launch_factor(sf.stream(), L.F, P, L.iota, L.B.gam, L.O, L.err);
      if (L.gam_s) {
        launch_scale_f64(sf.stream(), L.gam_s, L.B.gam, P, ctx->opt.scan_gamma_factor);
        launch_factor(sf.stream(), L.Fs, P, L.iota, L.gam_s, L.O, L.err);
      }
      launch_burgers_source(st, P, s, n, nu, u0, L.Uk, L.ubar, f, L.G);
      std::vector<int> me(E);
      int mmax = svd_stage(st, L.S, &L.B, E, n, s, L.G, tau, eta, h, me.data());
      sf.join();
      int herr = 0;
      PEXP_CUDA_TRY(cudaMemcpyAsync(&herr, L.err, sizeof(int), cudaMemcpyDeviceToHost, st));
      host_sync(st);
      if (herr) fail(PEXP_EPIVOT, "shift-and-invert factorisation: a pivot is zero relative to its row or non-finite");
      max_m = std::max(max_m, mmax);
      if (rec_m) std::copy(me.begin(), me.end(), rec_m + size_t(k) * P);
      if (rec_g) PEXP_CUDA_TRY(cudaMemcpyAsync(rec_g + size_t(k) * P, L.B.gam, P * sizeof(double),
                                               cudaMemcpyDeviceToHost, st));
      launch_fill_i32(st, L.B.krec, E, 0);
      g_cfg.kprev = k > 0 ? kprev.data() : nullptr;
      if (mmax > 0) {
        RunInfo ri = ebk_forced(st, L.B, L.S, L.F, L.O, true, E, mmax, me.data(), h, s, 1, s, 0, L.Y, (long long)s * n,
                                        o.stop_rule, o.restart_blocks);
        if (ri.unconverged) fail(PEXP_ENOCONV, "Krylov capacity reached (nonhomogeneous, WR iteration " + std::to_string(k + 1) + ")");
        max_k = std::max(max_k, ri.max_ktot);
        restarts += ri.restarts;
      } else {
        PEXP_CUDA_TRY(cudaMemsetAsync(L.Y, 0, size_t(P) * s * n * sizeof(double), st));
      }
      if (rec_k) PEXP_CUDA_TRY(cudaMemcpyAsync(rec_k + size_t(k) * P, L.B.krec, P * sizeof(int),
                                               cudaMemcpyDeviceToHost, st));
      // read back with the delta synchronisation below: the next iteration's check-schedule hint
      PEXP_CUDA_TRY(cudaMemcpyAsync(kcur.data(), L.B.krec, P * sizeof(int), cudaMemcpyDeviceToHost, st));
      PEXP_CUDA_TRY(cudaMemsetAsync(L.delta, 0, sizeof(double), st));
      scan_ev.emplace_back(new EventPair);
      PEXP_CUDA_TRY(cudaEventRecord(scan_ev.back()->a, st));
      if (L.scan_ws) {  // persistent cooperative scan; host-driven fallback beyond its row capacity
        const int k1 = std::min(o.kcap, 512);
        const double defl_s = g_cfg.defl;
        max_k = std::max(max_k, launch_hom_scan(st, L.gam_s ? L.Fs : L.F, L.gam_s ? L.gam_s : L.B.gam, P, s, n, k1, h,
                                                eta, defl_s, u0, L.Y, L.Uk, L.Un,
                                                L.delta, L.scan_ws, L.scan_bytes,
                                                rec_ks ? rec_ks + size_t(k) * P : nullptr, scan_diag));
      } else
      for (int i = 0; i < P; ++i) {
        const size_t off = size_t(i) * s * n;
        if (i == 0) {
          launch_wr_step(st, s, n, u0, nullptr, L.Y + off, L.Uk + off, L.Un + off, L.uhat, L.delta);
          continue;
        }
        // homogeneous scan step: exp((t - T_{i-1}) A_i) uhat(T_{i-1}) at the s nodes
        EbkBufs& B1 = L.B1;
        k_hom_start<<<1, PEXP_THREADS, 0, st>>>(2, n, L.uhat, n, B1.beta, B1.V, B1.vs_e);
        count_launch();
        PEXP_CUDA_TRY(cudaMemcpyAsync(B1.fidx, L.iota + i, sizeof(int), cudaMemcpyDeviceToDevice, st));
        PEXP_CUDA_TRY(cudaMemcpyAsync(B1.opidx, L.iota + i, sizeof(int), cudaMemcpyDeviceToDevice, st));
        PEXP_CUDA_TRY(cudaMemcpyAsync(B1.gam, L.B.gam + i, sizeof(double), cudaMemcpyDeviceToDevice, st));
        launch_hom_setup(st, 1, 1, P, s, h, eta, B1.beta, B1.crit, B1.npieces, B1.active);
        RunInfo rh = ebk_run(st, B1, L.F, L.O, true, 1, 1, h, 0, 1, s, o.stop_rule);
        if (rh.unconverged) fail(PEXP_ENOCONV, "Krylov capacity reached (homogeneous scan)");
        max_k = std::max(max_k, rh.max_k);
        launch_combine(st, 1, n, B1.V, B1.vs_e, 0, std::max(rh.max_k, 1), B1.Z, B1.zs_e, B1.kcap, L.Wh, (long long)s * n, 0, s,
                       1.0, 0.0, nullptr, B1.kfin);
        launch_wr_step(st, s, n, u0, L.Wh, L.Y + off, L.Uk + off, L.Un + off, L.uhat, L.delta);
      }
      PEXP_CUDA_TRY(cudaEventRecord(scan_ev.back()->b, st));
      PEXP_CUDA_TRY(cudaMemcpyAsync(&delta, L.delta, sizeof(double), cudaMemcpyDeviceToHost, st));
      host_sync(st);
      std::swap(L.Uk, L.Un);
      kprev = kcur;
      dhist.push_back(delta);
      ++iters;
      if (delta0 < 0) delta0 = delta;
      if (!std::isfinite(delta) || delta > 1e3 * delta0)
        fail(PEXP_EDIVERGED, "waveform relaxation diverged at iteration " + std::to_string(iters));
      if (delta < wr_tol) break;
    }
    launch_copy_end(st, P, s, n, L.Uk, out);
    if (Uout) PEXP_CUDA_TRY(cudaMemcpyAsync(Uout, L.Uk, size_t(P) * s * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    PEXP_CUDA_TRY(cudaEventRecord(ev.b, st));
    PEXP_CUDA_TRY(cudaEventSynchronize(ev.b));
    ++g_cfg.syncs;
    const float ms = ev.ms();
    check_err(st);
    if (st_out) {
      std::memset(st_out, 0, sizeof(*st_out));
      st_out->m_j = rec_m; st_out->k_j = rec_k; st_out->gamma_j = rec_g; st_out->kscan_j = rec_ks;
      for (int q = 0; q < std::min<int>(iters, 64); ++q) st_out->delta_hist[q] = dhist[q];
      st_out->host_syncs = g_cfg.syncs;
      st_out->wr_iters = iters;
      st_out->wr_last_delta = delta;
      st_out->max_m = max_m;
      st_out->max_k = max_k;
      st_out->restarts = restarts;
      st_out->ms_total = ms;
      for (auto& e : scan_ev) st_out->ms_hom += e->ms();
      st_out->scan_steps = scan_diag[0];
      st_out->scan_checks = scan_diag[1];
      st_out->scan_check_cycles = scan_diag[2];
      st_out->ms_nonhom = ms - st_out->ms_hom;
      st_out->evals = P * iters;
      st_out->kernel_launches = (int)g_launches;
    }
  });
}

pexp_status pexp_sai_solve(pexp_ctx* ctx, int32_t b, double gamma, const double* rhs, int32_t ncols, double* x) {
  if (!ctx) return PEXP_EINVAL;
  if (b < 0 || b >= ctx->batch || !(gamma > 0) || ncols < 0 || !rhs || !x) return set_err(ctx, PEXP_EINVAL, "bad argument");
  if (!ctx->ws || ctx->ws_bytes < lin_bytes(ctx, 1)) return set_err(ctx, PEXP_ENOMEM, "workspace not set or too small");
  return guarded(ctx, [&] {
    init_once();
    Opts o = norm_opts(ctx->opt);
    g_cfg = o.cfg;
    cudaStream_t st = o.st;
    const int n = (int)ctx->n;
    Arena ar{ctx->ws, ctx->ws_bytes, 0};
    LinPlan L;
    plan_linear(ar, L, ctx, 1);
    std::vector<double> nu1{ctx->nu[b]}, a1{ctx->a[b]}, g1{gamma};
    std::vector<int> z1{0};
    h2d(st, L.nu_d, nu1);
    h2d(st, L.a_d, a1);
    h2d(st, L.gam_f, g1);
    h2d(st, L.opidx_f, z1);
    Ops O1 = L.O;
    O1.nops = 1;
    launch_ade_rows(st, 1, n, ctx->bc == PEXP_BC_DIRICHLET, L.nu_d, L.a_d, O1.sub, O1.diag, O1.sup);
    PEXP_CUDA_TRY(cudaMemsetAsync(L.err, 0, sizeof(int), st));
    launch_factor(st, L.F, 1, L.opidx_f, L.gam_f, O1, L.err);
    launch_sai_solve(st, L.F, nullptr, 1, ncols, rhs, 0, 0, x, 0, 0, nullptr, nullptr, 0);
    int herr = 0;
    PEXP_CUDA_TRY(cudaMemcpyAsync(&herr, L.err, sizeof(int), cudaMemcpyDeviceToHost, st));
    host_sync(st);
    if (herr) fail(PEXP_EPIVOT, "shift-and-invert factorisation: a pivot is zero relative to its row or non-finite");
  });
}

pexp_status pexp_source_svd(pexp_ctx* ctx, const double* G, int32_t E, double tol, int32_t* m_host, double* sigma,
                            double* proj) {
  if (!ctx) return PEXP_EINVAL;
  if (!G || !m_host || !sigma || !proj || E < 1) return set_err(ctx, PEXP_EINVAL, "bad argument");
  if (!(tol >= 1e-14 && tol <= 1e-2)) return set_err(ctx, PEXP_EINVAL, "tol must be in [1e-14, 1e-2]");
  Opts o0 = norm_opts(ctx->opt);
  int Pneed = (E + ctx->batch - 1) / ctx->batch;
  if (!ctx->ws || ctx->ws_bytes < lin_bytes(ctx, Pneed)) return set_err(ctx, PEXP_ENOMEM, "workspace too small");
  (void)o0;
  return guarded(ctx, [&] {
    init_once();
    Opts o = norm_opts(ctx->opt);
    g_cfg = o.cfg;
    cudaStream_t st = o.st;
    const int n = (int)ctx->n, s = o.s;
    Arena ar{ctx->ws, ctx->ws_bytes, 0};
    LinPlan L;
    plan_linear(ar, L, ctx, Pneed);
    L.B.E = E;
    const double tau = o.tau_f * tol;
    int mmax = svd_stage(st, L.S, &L.B, E, n, s, G, tau, o.eta_f * tol, 1.0, m_host);
    PEXP_CUDA_TRY(cudaMemcpyAsync(sigma, L.S.sig, size_t(E) * s * sizeof(double), cudaMemcpyDeviceToDevice, st));
    int mb = std::max(mmax, 1);
    launch_combine(st, E, n, L.S.U, (long long)s * n, 0, mb, L.S.Cfin, (long long)mb * s, mb, proj, (long long)s * n, 0,
                   s, 1.0, 0.0, nullptr);
    host_sync(st);
  });
}

pexp_status pexp_expm_batched(pexp_ctx* ctx, const double* A, int32_t E, int32_t N, double* X) {
  if (!ctx) return PEXP_EINVAL;
  if (!A || !X || E < 1 || N < 1 || N > 1024) return set_err(ctx, PEXP_EINVAL, "bad argument");
  const int nslots = std::min(E, 148);
  const size_t need = size_t(nslots) * (7ull * N * N * sizeof(double) + N * sizeof(int)) + 1024;
  if (!ctx->ws || ctx->ws_bytes < need) return set_err(ctx, PEXP_ENOMEM, "workspace too small for expm");
  return guarded(ctx, [&] {
    init_once();
    Opts o = norm_opts(ctx->opt);
    Arena ar{ctx->ws, ctx->ws_bytes, 0};
    double* work = ar.take<double>(size_t(nslots) * 7 * N * N);
    int* iwork = ar.take<int>(size_t(nslots) * N);
    launch_expm_batched(o.st, E, N, A, X, work, 7LL * N * N, iwork, nslots);
    host_sync(o.st);
  });
}

void pexp_profile_enable(int32_t on) {
  for (auto& r : g_prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  g_prof.clear();
  g_prof_on = on != 0;
}

int32_t pexp_profile_read(int32_t ncat, double* ms, double* bytes, double* flops, int32_t* launches) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  for (int c = 0; c < ncat; ++c) { ms[c] = 0; bytes[c] = 0; flops[c] = 0; launches[c] = 0; }
  for (auto& r : g_prof) {
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.cat < ncat) { ms[r.cat] += t; bytes[r.cat] += r.bytes; flops[r.cat] += r.flops; launches[r.cat] += 1; }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  return PC_NCAT;
}

}  // extern "C"
