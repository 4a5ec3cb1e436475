// stencil.cu — subsystem (5): stencil / nonlinear-term kernels, source assembly,
// superposition and the waveform-relaxation update (all HBM-streaming, coalesced along n).
#include "common.cuh"
#include "kernels.cuh"

namespace pexp {

// Y[e][y0+c] = A_op X[e][x0+c]   (tridiagonal rows; periodic wrap or zero Dirichlet values)
__global__ void k_apply_A(int n, const double* sub, const double* diag, const double* sup, const int* opidx,
                          const double* gam, const double* X, long long xs_e, int x0, double* Y,
                          long long ys_e, int y0, int periodic, int shifted, const int* active) {
  const int c = blockIdx.y, e = blockIdx.z;
  if (active && !active[e]) return;
  const size_t o = size_t(opidx ? opidx[e] : e) * n;
  const double* x = X + e * xs_e + size_t(x0 + c) * n;
  double* y = Y + e * ys_e + size_t(y0 + c) * n;
  const double g = shifted ? gam[e] : 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double xm = i > 0 ? x[i - 1] : (periodic ? x[n - 1] : 0.0);
    double xp = i < n - 1 ? x[i + 1] : (periodic ? x[0] : 0.0);
    double ax = sub[o + i] * xm + diag[o + i] * x[i] + sup[o + i] * xp;
    y[i] = shifted ? x[i] - g * ax : ax;
  }
}

// G[b][j][i][r] = Au0[b][r] + src[b][j][i][r]   (Eq.(linivp_shift))
__global__ void k_lin_source(long long total, int P, int s, int n, const double* Au0, const double* src,
                             double* G) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    long long r = k % n;
    long long b = k / ((long long)P * s * n);
    G[k] = Au0[b * n + r] + src[k];
  }
}

__device__ __forceinline__ double hash_uniform(unsigned e, unsigned c, unsigned r, unsigned seed) {
  unsigned long long x = (unsigned long long)e * 0x9E3779B97F4A7C15ull ^ ((unsigned long long)c << 32) ^ r ^
                         ((unsigned long long)seed << 17);
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

// V[e][c] <- pseudo-random where fill[e*mmax+c] (padding columns of the first Krylov block)
__global__ void k_fill_random(int n, int mmax, const int* fill, double* V, long long vs_e, unsigned seed) {
  const int c = blockIdx.y, e = blockIdx.z;
  if (!fill[e * mmax + c]) return;
  double* v = V + e * vs_e + size_t(c) * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[i] = hash_uniform(e, c, i, seed);
}

__global__ void k_broadcast(long long total, int n, const double* u0, double* U) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x)
    U[k] = u0[k % n];
}

// ubar_j = (1/(s-1)) [u_0/2 + u_1 + ... + u_{s-2} + u_{s-1}/2]  (trapezoid mean, reading #3)
__global__ void k_ubar(int s, int n, const double* U, double* ubar) {
  const int j = blockIdx.y;
  const double* Uj = U + size_t(j) * s * n;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double a = 0.5 * (Uj[r] + Uj[size_t(s - 1) * n + r]);
    for (int i = 1; i < s - 1; ++i) a += Uj[size_t(i) * n + r];
    ubar[size_t(j) * n + r] = a / (s - 1);
  }
}

// gamma_j = min(g0, 0.5 / max_r(-(D1 ubar_j)_r)), g0 = gamma_factor dT/10  (reading #4; keeps pivot-free solves safe)
__global__ void k_gamma(int n, const double* ubar, double g0, double* gam) {
  const int j = blockIdx.x;
  __shared__ double red[32];
  const double* u = ubar + size_t(j) * n;
  const double inv2dx = 0.5 * n;
  double mx = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    int rm = r == 0 ? n - 1 : r - 1, rp = r == n - 1 ? 0 : r + 1;
    mx = fmax(mx, -(u[rp] - u[rm]) * inv2dx);
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) {
    double g = g0;
    if (mx > 0.0) g = fmin(g, 0.5 / mx);
    gam[j] = g;
  }
}

// Shifted WR source at the nodes (Eq.(sourceParallel) PAPER.md:312 with reading #2):
//   G = nu D2 u0 - u∘D1u - J(ubar)(u - u0),  J(ubar) v = -(D1 ubar)∘v - ubar∘(D1 v)
// f (nullable): forcing samples f(x, t_{j,i}) of Eq.(burgersEq), [P][s][n]
__global__ void k_burgers_source(int s, int n, double nu, const double* u0, const double* U, const double* ubar,
                                 const double* f, double* G) {
  const int i = blockIdx.y, j = blockIdx.z;
  const double* u = U + (size_t(j) * s + i) * n;
  const double* ub = ubar + size_t(j) * n;
  double* g = G + (size_t(j) * s + i) * n;
  const double dx2 = double(n) * double(n), inv2dx = 0.5 * n;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    int rm = r == 0 ? n - 1 : r - 1, rp = r == n - 1 ? 0 : r + 1;
    double d2u0 = (u0[rm] - 2.0 * u0[r] + u0[rp]) * dx2;
    double d1u = (u[rp] - u[rm]) * inv2dx;
    double d1ub = (ub[rp] - ub[rm]) * inv2dx;
    double v = u[r] - u0[r], vm = u[rm] - u0[rm], vp = u[rp] - u0[rp];
    double d1v = (vp - vm) * inv2dx;
    double gv = nu * d2u0 - u[r] * d1u + d1ub * v + ub[r] * d1v;
    if (f) gv += f[(size_t(j) * s + i) * n + r];
    g[r] = gv;
  }
}

// One scan step of the WR update on subinterval i (Eq.(updateSolution)):
//   Unew[q] = u0 + Wh[q] + Y[q] at the s nodes; uhat_end = Wh[s-1] + Y[s-1];
//   delta = max(delta, max|Unew - Uold|)
__global__ void k_wr_step(int s, int n, const double* u0, const double* Wh, const double* Y, const double* Uold,
                          double* Unew, double* uhat_end, double* delta) {
  __shared__ double red[32];
  double mx = 0.0;
  const long long total = (long long)s * n;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    int r = int(k % n);
    int q = int(k / n);
    double uh = Y[k] + (Wh ? Wh[k] : 0.0);
    double un = u0[r] + uh;
    mx = fmax(mx, fabs(un - Uold[k]));
    if (!isfinite(un)) mx = INFINITY;
    Unew[k] = un;
    if (q == s - 1) uhat_end[r] = uh;
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) atomic_max_nonneg(delta, mx);
}

// out[b][i] = u0[b] + Yend[b*P+i] + sum_g Yh[b*groups+g][i]   (Eq.(superposition) PAPER.md:226;
// Yh[.][i] already sums the legs of group g that reach T_{i+1})
__global__ void k_superpose(int P, int n, const double* u0, const double* Yend, const double* Yh, long long yh_e,
                            long long yh_node, int groups, double* out) {
  const int i = blockIdx.y, b = blockIdx.z;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double a = u0[size_t(b) * n + r] + Yend[(size_t(b) * P + i) * n + r];
    if (Yh)
      for (int g = 0; g < groups; ++g) a += Yh[(long long)(b * groups + g) * yh_e + i * yh_node + r];
    out[(size_t(b) * P + i) * n + r] = a;
  }
}

// Grouped legs: column c of group eh = b*groups + g starts from v_j(T_{j+1}) = Y[b*P + j],
// j = g*mh + c (zero column when j >= P-1); beta = its norm.
__global__ void k_hom_start_block(int mh, int groups, int P, int n, const double* Y, double* V, long long vs_e,
                                  double* beta) {
  const int eh = blockIdx.x, c = blockIdx.y;
  __shared__ double red[32];
  const int b = eh / groups, g = eh % groups, j = g * mh + c;
  double* v = V + eh * vs_e + size_t(c) * n;
  const bool ok = j < P - 1;
  const double* y = Y + (size_t(b) * P + (ok ? j : 0)) * n;
  double a = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double x = ok ? y[r] : 0.0;
    v[r] = x;
    a = fma(x, x, a);
  }
  a = block_sum(a, red);
  if (threadIdx.x == 0) beta[size_t(eh) * mh + c] = sqrt(a);
}

__global__ void k_hom_setup_block(int Eh, int mh, int groups, int P, double dT, double eta, const double* beta,
                                  double* critc, int* horc, int* active) {
  for (int eh = blockIdx.x * blockDim.x + threadIdx.x; eh < Eh; eh += gridDim.x * blockDim.x) {
    const int g = eh % groups;
    int any = 0;
    for (int c = 0; c < mh; ++c) {
      const int j = g * mh + c;
      const double bt = beta[size_t(eh) * mh + c];
      const int hor = (j < P - 1 && bt > 0.0) ? (P - 1 - j) : 0;
      horc[size_t(eh) * mh + c] = hor;
      critc[size_t(eh) * mh + c] = hor > 0 ? eta * bt / (hor * dT) : 1.0;
      any |= hor > 0;
    }
    active[eh] = any;
  }
}

__global__ void k_copy_end(int s, int n, const double* U, double* out) {
  const int j = blockIdx.y;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    out[size_t(j) * n + r] = U[(size_t(j) * s + s - 1) * n + r];
}

__global__ void k_norms(int n, const double* X, long long xs_e, double* nrm) {
  const int e = blockIdx.x;
  __shared__ double red[32];
  const double* x = X + e * xs_e;
  double a = 0.0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) a = fma(x[r], x[r], a);
  a = block_sum(a, red);
  if (threadIdx.x == 0) nrm[e] = sqrt(a);
}

__global__ void k_scale_cols(int n, const double* X, long long xs_e, const double* nrm, double* Y, long long ys_e) {
  const int e = blockIdx.y;
  const double s = nrm[e] > 0.0 ? 1.0 / nrm[e] : 0.0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    Y[e * ys_e + r] = X[e * xs_e + r] * s;
}

// D_e[0:rows, 0:cols] += S_e[0:rows, 0:cols]
__global__ void k_add_block(int rows, int cols, const double* S, long long ss_e, int lds, double* D, long long ds_e,
                            int ldd, const int* active) {
  const int e = blockIdx.y;
  if (active && !active[e]) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < rows * cols; k += gridDim.x * blockDim.x) {
    int i = k % rows, j = k / rows;
    D[e * ds_e + i + size_t(j) * ldd] += S[e * ss_e + i + size_t(j) * lds];
  }
}

// H_e[0:rows, 0:m] += T_e[0:rows, 0:m] * R_e (m x m, general: pivoted CholQR factors)
__global__ void k_hupdate(int rows, int m, const double* T, long long ts_e, int ldt, const double* R, long long rs_e,
                          int ldr, double* H, long long hs_e, int ldh, const int* active) {
  const int e = blockIdx.y;
  if (active && !active[e]) return;
  const double* Te = T + e * ts_e;
  const double* Re = R + e * rs_e;
  double* He = H + e * hs_e;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < rows * m; k += gridDim.x * blockDim.x) {
    int i = k % rows, j = k / rows;
    double a = 0.0;
    for (int p = 0; p < m; ++p) a = fma(Te[i + size_t(p) * ldt], Re[p + size_t(j) * ldr], a);
    He[i + size_t(j) * ldh] += a;
  }
}

// Homogeneous legs: mode 0 = linear leg of eval (b, j) over [T_{j+1}, T_P] (npieces =
// (P-1-j)(s-1)); mode 1 = one scan step over one subinterval (npieces = s-1).
// crit = eta * beta / horizon; inactive when beta == 0.
__global__ void k_hom_setup(int E, int mode, int P, int s, double h, double eta, const double* beta, double* crit,
                            int* npieces, int* active) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    int np = mode == 0 ? (P - 1 - e % (P - 1)) * (s - 1) : (s - 1);
    npieces[e] = np;
    crit[e] = eta * beta[e] / (np * h);
    active[e] = beta[e] > 0.0;
  }
}

__global__ void k_update_active(int E, const int* conv, int* active, int* count, int* krec, int kval) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    if (active[e] && conv[e]) {
      active[e] = 0;
      if (krec) krec[e] = kval;  // total Krylov dimension at convergence (pexp_stats.k_j)
    }
    if (active[e]) atomicAdd(count, 1);
  }
}

__global__ void k_fill_i32(int* p, int count, int v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) p[i] = v;
}
__global__ void k_fill_f64(double* p, size_t count, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_scale_f64(double* y, const double* x, int n, double f) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = f * x[i];
}
void launch_scale_f64(cudaStream_t st, double* y, const double* x, int n, double f) {
  k_scale_f64<<<cdiv(n, 256), 256, 0, st>>>(y, x, n, f);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- width buckets (pexp_api.cu)
// Gather evaluations perm[0..ec) into the slots of one EBK chunk of block width wb: per-eval
// scalars, the first wb columns of the orthonormal source basis (basis block 0) and the first wb
// coefficient rows of the piecewise polynomial p(t) (layout [s-1][nq][w], w = mmax -> wb).
__global__ void k_bucket_gather(GatherArgs a) {
  const int i = blockIdx.y, e = a.perm[i];
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      a.gam_c[i] = a.gam[e];
      a.crit_c[i] = a.crit[e];
      a.active_c[i] = a.active[e];
      a.fidx_c[i] = a.fidx[e];
      a.opidx_c[i] = a.opidx[e];
    }
    const int np = (a.s - 1) * a.nq;
    for (int idx = threadIdx.x; idx < np * a.wb; idx += blockDim.x) {
      const int pq = idx / a.wb, c = idx % a.wb;
      a.coef_c[size_t(i) * np * a.wb + idx] = a.coef[size_t(e) * np * a.mmax + size_t(pq) * a.mmax + c];
    }
  }
  const size_t cnt = size_t(a.wb) * a.n;
  const double* src = a.U + e * a.us_e;
  double* dst = a.V + i * a.vs_e;
  for (size_t k = size_t(blockIdx.x) * blockDim.x + threadIdx.x; k < cnt; k += size_t(gridDim.x) * blockDim.x)
    dst[k] = src[k];
}

// Outputs of chunk slot i (cnt doubles at Yt + i*yts) back to evaluation perm[i] (Y + e*ys_e),
// and the slot's Krylov-dimension record.
__global__ void k_bucket_scatter(const int* perm, size_t cnt, const double* Yt, long long yts, double* Y,
                                 long long ys_e, const int* krec_c, int* krec) {
  const int i = blockIdx.y, e = perm[i];
  if (blockIdx.x == 0 && threadIdx.x == 0 && krec) krec[e] = krec_c[i];
  const double* src = Yt + i * yts;
  double* dst = Y + e * ys_e;
  for (size_t k = size_t(blockIdx.x) * blockDim.x + threadIdx.x; k < cnt; k += size_t(gridDim.x) * blockDim.x)
    dst[k] = src[k];
}

void launch_bucket_gather(cudaStream_t st, int ec, const GatherArgs& a) {
  if (ec == 0) return;
  ProfScope ps(PC_STENCIL, st, double(ec) * a.wb * a.n * 16.0, 0.0);
  dim3 grid(std::max(1, std::min(cdiv(long(a.wb) * a.n, 4 * PEXP_THREADS), 64)), ec);
  k_bucket_gather<<<grid, PEXP_THREADS, 0, st>>>(a);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_bucket_scatter(cudaStream_t st, int ec, const int* perm, size_t cnt, const double* Yt, long long yts,
                           double* Y, long long ys_e, const int* krec_c, int* krec) {
  if (ec == 0) return;
  ProfScope ps(PC_STENCIL, st, double(ec) * cnt * 16.0, 0.0);
  dim3 grid(std::max(1, std::min(cdiv(long(cnt), 4 * PEXP_THREADS), 64)), ec);
  k_bucket_scatter<<<grid, PEXP_THREADS, 0, st>>>(perm, cnt, Yt, yts, Y, ys_e, krec_c, krec);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- host wrappers
static int gx(long long n) { return int(std::min<long long>((n + PEXP_THREADS - 1) / PEXP_THREADS, 4096)); }
static int gx_small(int n, int others) {
  // enough CTAs along n so that the whole grid has >= ~4 waves
  int g = cdiv(n, PEXP_THREADS);
  int want = std::max(1, (148 * 8) / std::max(1, others));
  return std::max(1, std::min(g, want));
}

void launch_apply_A(cudaStream_t st, const Ops& O, const int* opidx, int E, int ncols, const double* X,
                    long long xs_e, int x0, double* Y, long long ys_e, int y0, bool periodic) {
  if (E == 0 || ncols == 0) return;
  dim3 grid(gx_small(O.n, E * ncols), ncols, E);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_apply_A<<<grid, PEXP_THREADS, 0, st>>>(O.n, O.sub, O.diag, O.sup, opidx, nullptr, X, xs_e, x0, Y, ys_e, y0,
                                            periodic, 0, nullptr);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_apply_M(cudaStream_t st, const Ops& O, const int* opidx, const double* gam, int E, int ncols,
                    const double* X, long long xs_e, int x0, double* Y, long long ys_e, int y0, bool periodic,
                    const int* active) {
  if (E == 0 || ncols == 0) return;
  dim3 grid(gx_small(O.n, E * ncols), ncols, E);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_apply_A<<<grid, PEXP_THREADS, 0, st>>>(O.n, O.sub, O.diag, O.sup, opidx, gam, X, xs_e, x0, Y, ys_e, y0,
                                            periodic, 1, active);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_lin_source(cudaStream_t st, int batch, int P, int s, int n, const double* Au0, const double* src,
                       double* G) {
  long long total = (long long)batch * P * s * n;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_lin_source<<<gx(total), PEXP_THREADS, 0, st>>>(total, P, s, n, Au0, src, G);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_fill_random(cudaStream_t st, int E, int n, int mmax, const int* fill, double* V, long long vs_e,
                        unsigned seed) {
  dim3 grid(gx_small(n, E * mmax), mmax, E);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_fill_random<<<grid, PEXP_THREADS, 0, st>>>(n, mmax, fill, V, vs_e, seed);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_broadcast_waveform(cudaStream_t st, int P, int s, int n, const double* u0, double* U) {
  long long total = (long long)P * s * n;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_broadcast<<<gx(total), PEXP_THREADS, 0, st>>>(total, n, u0, U);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_ubar_gamma(cudaStream_t st, int P, int s, int n, const double* U, double g0, double* ubar,
                       double* gam) {
  dim3 grid(gx_small(n, P), P);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_ubar<<<grid, PEXP_THREADS, 0, st>>>(s, n, U, ubar);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_gamma<<<P, PEXP_THREADS, 0, st>>>(n, ubar, g0, gam);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_burgers_source(cudaStream_t st, int P, int s, int n, double nu, const double* u0, const double* U,
                           const double* ubar, const double* f, double* G) {
  dim3 grid(gx_small(n, P * s), s, P);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_burgers_source<<<grid, PEXP_THREADS, 0, st>>>(s, n, nu, u0, U, ubar, f, G);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_wr_step(cudaStream_t st, int s, int n, const double* u0, const double* Wh, const double* Y,
                    const double* Uold, double* Unew, double* uhat_end, double* delta) {
  long long total = (long long)s * n;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_wr_step<<<std::min(gx(total), 592), PEXP_THREADS, 0, st>>>(s, n, u0, Wh, Y, Uold, Unew, uhat_end, delta);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_superpose(cudaStream_t st, int batch, int P, int n, const double* u0, const double* Yend,
                      const double* Yh, long long yh_e, long long yh_node, int groups, double* out) {
  dim3 grid(gx_small(n, batch * P), P, batch);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_superpose<<<grid, PEXP_THREADS, 0, st>>>(P, n, u0, Yend, Yh, yh_e, yh_node, groups, out);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_copy_end(cudaStream_t st, int P, int s, int n, const double* U, double* out) {
  dim3 grid(gx_small(n, P), P);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_copy_end<<<grid, PEXP_THREADS, 0, st>>>(s, n, U, out);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_norms(cudaStream_t st, int E, int n, const double* X, long long xs_e, double* nrm) {
  if (E == 0) return;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_norms<<<E, PEXP_THREADS, 0, st>>>(n, X, xs_e, nrm);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_scale_cols(cudaStream_t st, int E, int n, const double* X, long long xs_e, const double* nrm,
                       double* Y, long long ys_e) {
  if (E == 0) return;
  dim3 grid(gx_small(n, E), E);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_scale_cols<<<grid, PEXP_THREADS, 0, st>>>(n, X, xs_e, nrm, Y, ys_e);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_add_block(cudaStream_t st, int E, int rows, int cols, const double* S, long long ss_e, int lds,
                      double* D, long long ds_e, int ldd, const int* active) {
  if (E == 0 || rows * cols == 0) return;
  dim3 grid(std::min(cdiv(rows * cols, PEXP_THREADS), 64), E);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_add_block<<<grid, PEXP_THREADS, 0, st>>>(rows, cols, S, ss_e, lds, D, ds_e, ldd, active);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_hupdate(cudaStream_t st, int E, int rows, int m, const double* T, long long ts_e, int ldt, const double* R,
                    long long rs_e, int ldr, double* H, long long hs_e, int ldh, const int* active) {
  if (E == 0 || rows * m == 0) return;
  dim3 grid(std::min(cdiv(rows * m, PEXP_THREADS), 64), E);
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_hupdate<<<grid, PEXP_THREADS, 0, st>>>(rows, m, T, ts_e, ldt, R, rs_e, ldr, H, hs_e, ldh, active);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_hom_start_block(cudaStream_t st, int Eh, int mh, int groups, int P, int n, const double* Y, double* V,
                            long long vs_e, double* beta) {
  if (Eh == 0) return;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_hom_start_block<<<dim3(Eh, mh), PEXP_THREADS, 0, st>>>(mh, groups, P, n, Y, V, vs_e, beta);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_hom_setup_block(cudaStream_t st, int Eh, int mh, int groups, int P, double dT, double eta,
                            const double* beta, double* critc, int* horc, int* active) {
  if (Eh == 0) return;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_hom_setup_block<<<cdiv(Eh, 128), 128, 0, st>>>(Eh, mh, groups, P, dT, eta, beta, critc, horc, active);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_hom_setup(cudaStream_t st, int E, int mode, int P, int s, double h, double eta, const double* beta,
                      double* crit, int* npieces, int* active) {
  if (E == 0) return;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_hom_setup<<<cdiv(E, PEXP_THREADS), PEXP_THREADS, 0, st>>>(E, mode, P, s, h, eta, beta, crit, npieces, active);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_update_active(cudaStream_t st, int E, const int* conv, int* active, int* count, int* krec, int kval) {
  if (E == 0) return;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_update_active<<<std::min(cdiv(E, PEXP_THREADS), 256), PEXP_THREADS, 0, st>>>(E, conv, active, count, krec, kval);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_fill_i32(cudaStream_t st, int* p, int count, int v) {
  if (count <= 0) return;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_fill_i32<<<std::min(cdiv(count, PEXP_THREADS), 1024), PEXP_THREADS, 0, st>>>(p, count, v);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_fill_f64(cudaStream_t st, double* p, size_t count, double v) {
  if (count == 0) return;
  { ProfScope ps(PC_STENCIL, st, 0.0, 0.0);
  k_fill_f64<<<int(std::min<size_t>((count + PEXP_THREADS - 1) / PEXP_THREADS, 4096)), PEXP_THREADS, 0, st>>>(p, count, v);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

}  // namespace pexp
