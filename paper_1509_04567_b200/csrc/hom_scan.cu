// hom_scan.cu — the Burgers homogeneous scan (Fig. 5 / Eq.
// (updateSolution) P:331-335) as ONE persistent cooperative kernel.
//
// For subinterval i = 1..P-1 (sequential: the operator A_i changes per subinterval):
//     u_hat(t) = exp((t - T_{i-1}) A_i) u_hat(T_{i-1}),   t = T_{i-1} + r h,  r = 0..s-1,
// by single-vector shift-and-invert Arnoldi on B_i = (I - gamma_i A_i)^{-1}, projected
// A_hat = (I - H^{-1}) / gamma_i, z(t) = exp(t A_hat) beta e_1, residual stop rule of DESIGN.md
// §3 #6 (SaI residual |h_{K+1,K} e_K^T H^{-1} z(t)| / gamma <= eta beta / dT).  The waveform
// update u_{k+1} = u0 + Y + u_hat and delta = max |u_{k+1} - u_k| (a7, a8) are fused in.
//
// Roles: CTAs 0..nw-1 are workers, each owning a contiguous segment of rows; CTA nw is the
// checker that solves the projected problem on the newest available Krylov dimension while the
// workers keep extending the basis (check latency overlaps the Arnoldi steps).  Worker 0 is the
// leader: it turns the checker's result into a decision that every worker reads after the next
// barrier, so all workers leave the Arnoldi loop at the same step.
//
// Per Arnoldi step (3 all-to-all exchanges between the workers, no barrier object):
//   A: forward L-solve maps of own rows (y affine in the carry-in cy), backward U-solve maps with
//      the offset kept affine in cy, Sherman-Morrison dot partial                    | exchange 1
//   B: every CTA composes all segments' maps (one warp): own carries cy, cx; y, x; SM correction;
//      CGS pass-1 dot partials                                                        | exchange 2
//   C: h = sum of partials; x -= V h; pass-2 dot partials and ||x||^2                 | exchange 3
//   D: h2; x -= V h2; ||x|| = sqrt(||x||^2 - ||h2||^2); v_{k+1}; H column; publish
// An exchange is a stamped all-gather through L2: every CTA stores its row of values into one of
// three rotating slots whose entries hold a sentinel (all-ones NaN pattern) until written; every
// CTA polls all rows (independent loads, all in flight) and sums them in a fixed order, so all
// CTAs hold bitwise identical results after ONE L2 round trip.  A CTA re-arms a slot's own row
// right after the gather two exchanges later (nobody can still be reading it, and the re-arm is
// fenced before its next publish).  The CTA's rows of the basis live in shared memory (the first
// vcap columns; later ones in L2), so the Gram-Schmidt passes never leave the SM.
#include <cstdlib>
#include "kernels.cuh"
#include "dense.cuh"
#include "scan.cuh"

namespace pexp {

namespace {

constexpr int RPT_MAX = 4;   // rows per thread
constexpr int NT = PEXP_THREADS;
constexpr int HS_PSM = 12288;  // checker's shared scratch (doubles) for the LU panel / permutation
constexpr int XG_DOUBLES = 148 * 8;  // gathered rows of exchange 1
// dynamic shared memory (doubles): hv, hv2, xs, then [xg | Vs] (workers) or the LU scratch (checker)
constexpr int SCAN_SMEM_DOUBLES = 26400;  // 206 KB dynamic (+ ~19 KB static of the dense helpers) of the 227 KB per CTA
constexpr int VS_DOUBLES = SCAN_SMEM_DOUBLES - 2 * (KSMALL_MAX + 8) - NT * RPT_MAX - XG_DOUBLES;
static_assert(XG_DOUBLES + VS_DOUBLES >= HS_PSM, "checker scratch must fit");
static_assert(SCAN_SMEM_DOUBLES >= 6 * 64 * 64 + 4 * 64, "small-matrix checker buffers must fit");

enum { F_STEPS = 0, F_RESULT = 1, F_DECISION = 2, F_KMAX = 3, F_ERR = 4, F_BREAK = 5,
       F_NSTEPS = 8, F_NCHECK = 9, F_CHKCYC = 10,  // diagnostics: Arnoldi steps, checks, checker kilo-cycles
       F_NFLAGS = 12 };
enum { B_WCNT = 0, B_WGEN = 1, B_ACNT = 2, B_AGEN = 3 };

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

// Sense-counting grid barrier over nb CTAs (co-residency guaranteed by the cooperative launch).
__device__ inline void gbar(unsigned* cnt, unsigned* gen, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = gen;
    const unsigned g0 = *vg;
    __threadfence();
    if (atomicAdd(cnt, 1u) == nb - 1) {
      atomicExch(cnt, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vg == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// Sum over CTAs of part[c*pw + j0 + j] for j < nval, in a fixed order; result to out[j] (smem).
// The NT threads form ng = NT / nval groups; group q sums CTAs q, q + ng, ... for its value j
// (independent loads, all in flight), the ng group partials are then summed in group order.  Every
// CTA computes the identical result.  out must hold >= NT doubles (scratch for the partials).
__device__ inline void grid_reduce(const double* part, int pw, int ncta, int j0, int nval, double* out) {
  if (nval <= 0) return;
  if (nval > NT / 2) {  // wide: one thread per value, CTAs in order
    for (int j = threadIdx.x; j < nval; j += NT) {
      double a = 0.0;
      for (int c = 0; c < ncta; ++c) a += __ldcg(part + size_t(c) * pw + j0 + j);
      out[j] = a;
    }
    __syncthreads();
    return;
  }
  const int ng = NT / nval;
  const int j = threadIdx.x % nval, q = threadIdx.x / nval;
  double a = 0.0;
  if (q < ng)
    for (int c = q; c < ncta; c += ng) a += __ldcg(part + size_t(c) * pw + j0 + j);
  __syncthreads();  // out may still be read by the caller's previous use
  if (q < ng) out[q * nval + j] = a;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < nval)
    for (int g = 0; g < ng; ++g) t += out[g * nval + threadIdx.x];
  __syncthreads();
  if (threadIdx.x < nval) out[threadIdx.x] = t;
  __syncthreads();
}

struct Aff3 {  // x -> A x + B0 + B1 cy  (offset affine in the forward carry-in cy)
  double A, B0, B1;
};
__device__ __forceinline__ Aff3 after3(Aff3 first, Aff3 then) {
  return {then.A * first.A, fma(then.A, first.B0, then.B0), fma(then.A, first.B1, then.B1)};
}

// Exclusive scan of Aff3 maps in REVERSE thread order (rank = NT - 1 - threadIdx.x), as
// block_excl_scan<true> of scan.cuh.
__device__ __forceinline__ Aff3 block_excl_scan3_rev(Aff3 v, int rank, Aff3* wsm, Aff3& total) {
  const int lane = rank & 31, w = rank >> 5;
  Aff3 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double pa = __shfl_down_sync(0xffffffffu, inc.A, o), p0 = __shfl_down_sync(0xffffffffu, inc.B0, o),
                 p1 = __shfl_down_sync(0xffffffffu, inc.B1, o);
    if (lane >= o) inc = after3(Aff3{pa, p0, p1}, inc);
  }
  const double ea = __shfl_down_sync(0xffffffffu, inc.A, 1), e0 = __shfl_down_sync(0xffffffffu, inc.B0, 1),
               e1 = __shfl_down_sync(0xffffffffu, inc.B1, 1);
  const Aff3 exc = lane == 0 ? Aff3{1.0, 0.0, 0.0} : Aff3{ea, e0, e1};
  __syncthreads();
  if (lane == 31) wsm[w] = inc;
  __syncthreads();
  if (rank == 0) {
    Aff3 acc{1.0, 0.0, 0.0};
    for (int k = 0; k < NT / 32; ++k) {
      const Aff3 t = wsm[k];
      wsm[k] = acc;
      acc = after3(acc, t);
    }
    wsm[NT / 32] = acc;
  }
  __syncthreads();
  const Aff3 pre = wsm[w];
  total = wsm[NT / 32];
  return after3(pre, exc);
}

// ---- stamped all-gather exchange (header comment)
__device__ __forceinline__ double ld_poll(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool is_sentinel(double v) { return __double_as_longlong(v) == -1LL; }
__device__ __forceinline__ double sentinel() { return __longlong_as_double(-1LL); }

struct Xch {
  double* base;  // [3][nw][pw]
  int nw, pw, c;
  int e = 0;               // exchange counter (identical in every worker)
  int lastn[3] = {0, 0, 0};  // values this CTA stored in each slot's row
  __device__ double* row(int slot, int cta) const { return base + (size_t(slot) * nw + cta) * pw; }
};

// Publish this CTA's nval values (shared memory src) in the current slot.  All threads call it.
__device__ inline void xch_publish(Xch& X, const double* src, int nval) {
  const int slot = X.e % 3;
  double* r = X.row(slot, X.c);
  for (int j = threadIdx.x; j < nval; j += NT) __stcg(r + j, src[j]);
  X.lastn[slot] = nval;
}

// After the gather of exchange e: re-arm the own row of slot (e + 2) % 3 and advance.
__device__ inline void xch_finish(Xch& X) {
  const int rs = (X.e + 2) % 3;
  double* r = X.row(rs, X.c);
  const int ln = X.lastn[rs];
  for (int j = threadIdx.x; j < ln; j += NT) __stcg(r + j, sentinel());
  X.lastn[rs] = 0;
  __threadfence();
  __syncthreads();
  ++X.e;
}

// Gather: out[cta * nval + j] for every CTA (nval small).  out in shared memory.
__device__ inline void xch_gather(Xch& X, int nval, double* out) {
  const int slot = X.e % 3;
  const int total = X.nw * nval;
  for (int i0 = threadIdx.x; i0 < total; i0 += 4 * NT) {
    double v[4];
    const double* p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * NT;
      p[u] = X.row(slot, (i < total ? i : 0) / nval) + (i < total ? i : 0) % nval;
      if (i < total) v[u] = ld_poll(p[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * NT;
      if (i < total) {
        while (is_sentinel(v[u])) v[u] = ld_poll(p[u]);
        out[i] = v[u];
      }
    }
  }
  xch_finish(X);
}

// Reduce: out[j] = sum over CTAs (fixed order: ng interleaved groups, then the groups in order) of
// value j, j < nval.  out (shared memory) must hold >= max(NT, nval) doubles.
__device__ inline void xch_reduce(Xch& X, int nval, double* out) {
  const int slot = X.e % 3;
  __syncthreads();  // out may be the publish source or still be read by the caller
  if (nval > NT / 2) {  // wide: one thread per value, CTAs in order
    for (int j = threadIdx.x; j < nval; j += NT) {
      double a = 0.0;
      for (int c0 = 0; c0 < X.nw; c0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + u < X.nw) v[u] = ld_poll(X.row(slot, c0 + u) + j);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + u < X.nw) {
            while (is_sentinel(v[u])) v[u] = ld_poll(X.row(slot, c0 + u) + j);
            a += v[u];
          }
      }
      out[j] = a;
    }
    xch_finish(X);
    return;
  }
  const int ng = NT / nval;
  const int j = threadIdx.x % nval, q = threadIdx.x / nval;
  double a = 0.0;
  if (q < ng) {
    for (int c0 = q; c0 < X.nw; c0 += 8 * ng) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + u * ng < X.nw) v[u] = ld_poll(X.row(slot, c0 + u * ng) + j);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + u * ng < X.nw) {
          while (is_sentinel(v[u])) v[u] = ld_poll(X.row(slot, c0 + u * ng) + j);
          a += v[u];
        }
    }
  }
  __syncthreads();  // out may still be read by the caller's previous use
  if (q < ng) out[q * nval + j] = a;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < nval)
    for (int g = 0; g < ng; ++g) t += out[g * nval + threadIdx.x];
  __syncthreads();
  if (threadIdx.x < nval) out[threadIdx.x] = t;
  xch_finish(X);
}

// Partial dots of the CTA's segment against basis columns 0..kk-1 (the first vcap from shared
// memory Vs, column stride segp; later ones from global Vg, column stride n) and ||x||^2:
// out[j] = V_j[seg] . x[seg] (j < kk), out[kk] = ||x[seg]||^2.  x staged in xs.
__device__ inline void seg_dots2(const double* Vs, int segp, int vcap, const double* Vg, int n, int row0, int nrow,
                                 int kk, const double* xr, int rpt, double* xs, double* out) {
  for (int q = 0; q < rpt; ++q) {
    const int l = threadIdx.x * rpt + q;
    if (l < nrow) xs[l] = xr[q];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = w; j <= kk; j += NT / 32) {
    double p0 = 0.0, p1 = 0.0;
    if (j < kk) {
      const double* v = j < vcap ? Vs + size_t(j) * segp : Vg + size_t(j) * n + row0;
      int l = lane;
      for (; l + 32 < nrow; l += 64) {
        p0 = fma(v[l], xs[l], p0);
        p1 = fma(v[l + 32], xs[l + 32], p1);
      }
      if (l < nrow) p0 = fma(v[l], xs[l], p0);
    } else {
      for (int l = lane; l < nrow; l += 32) p0 = fma(xs[l], xs[l], p0);
    }
    const double p = warp_sum(p0 + p1);
    if (lane == 0) out[j] = p;
  }
  __syncthreads();
}

}  // namespace

struct ScanArgs {
  int P, s, n, nw, seg, rpt, kcap, periodic;
  const double *fl, *fdinv, *fsup, *fz, *fw;  // factors, factor index = subinterval
  const double* gam;                          // [P]
  double h, eta, defl;
  const double *u0, *Y, *Uold;  // u0 [n]; Y, Uold [P][s][n]
  double* Unew;                 // [P][s][n]
  double* delta;                // max |Unew - Uold| (atomic max)
  double* V;                    // [kcap + 1][n]  scratch basis (subintervals not archived)
  double* H;                    // (kcap + 1) x kcap, ld kcap + 1
  double* Zc;                   // [P][s][kcap]   projected solutions at the nodes (per subinterval)
  double* Vpool;                // [pool_cols][n] archived bases (outputs computed after the scan)
  long long pool_cols;
  int* koff;                    // [P] pool column offset of subinterval i (-1: not archived)
  int* kc;                      // [P] converged dimension (-1: outputs written inside the scan)
  double* partA;                // [nw][pw]
  double* partB;                // [nw][pw]
  double* maps;                 // [2][nw][2]
  double* xch;                  // [3][nw][kcap + 8] exchange slots (sentinel-initialised)
  int vcap, segp;               // basis columns resident in shared memory; their column stride
  double* work;                 // checker: 10 kcap^2
  int* iwork;                   // checker: kcap
  unsigned* bar;                // [4]
  int* flags;                   // [F_NFLAGS]
};

// ---------------------------------------------------------------- small dense kit (checker CTA)
// K <= 64 (the usual scan space): the whole projected check runs out of shared memory -- six 64 x 64
// column-major buffers (ld SLD), zero-padded so the products need no bounds checks.
constexpr int SLD = 64;
constexpr int SMAT = SLD * SLD;

// C = A * B on the zero-padded 64 x 64 buffers, contraction over the first Np indices (Np = N rounded up
// to 4; C must not alias A or B).  Thread t owns rows (t % 16) + 16 ii and columns (t / 16) + 16 jj
// (conflict-free shared-memory reads: 16 consecutive doubles of A, broadcast of B).
__device__ inline void sm_gemm(int Np, const double* A, const double* B, double* C) {
  const int ti = threadIdx.x & 15, tj = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = 0.0;
  for (int k = 0; k < Np; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) av[ii] = A[ti + 16 * ii + k * SLD];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) bv[jj] = B[k + (tj + 16 * jj) * SLD];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = fma(av[ii], bv[jj], acc[ii][jj]);
  }
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) C[ti + 16 * ii + (tj + 16 * jj) * SLD] = acc[ii][jj];
  __syncthreads();
}

// Gauss-Jordan with partial (row) pivoting: M X = B solved in place (M destroyed, B <- X), N x N with
// nb right-hand columns.  col: N doubles of scratch.  Returns false on a zero pivot.
__device__ inline bool sm_gauss_jordan(int N, double* M, double* B, int nb, double* col, int* s_p) {
  for (int k = 0; k < N; ++k) {
    if (threadIdx.x < 32) {  // pivot row: largest |M[i][k]|, i >= k (first on ties)
      double best = -1.0;
      int bi = k;
      for (int i = k + threadIdx.x; i < N; i += 32) {
        const double v = fabs(M[i + k * SLD]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (threadIdx.x == 0) *s_p = best > 0.0 ? bi : -1;
    }
    __syncthreads();
    const int pr = *s_p;
    if (pr < 0) return false;
    // swap rows k <-> pr, scale row k by 1 / pivot (columns j >= k of M, all of B)
    const double pinv = 1.0 / M[pr + k * SLD];
    __syncthreads();
    for (int j = threadIdx.x; j < N + nb; j += NT) {
      double* X = j < N ? M + j * SLD : B + (j - N) * SLD;
      if (j < N && j < k) continue;
      const double a = X[pr], b = X[k];
      X[pr] = b;
      X[k] = a * pinv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += NT) col[i] = i == k ? 0.0 : M[i + k * SLD];
    __syncthreads();
    // eliminate column k from every other row
    for (int idx = threadIdx.x; idx < N * (N - k + nb); idx += NT) {
      const int i = idx % N, jj = idx / N;
      const int j = k + jj;  // k..N-1: M columns; beyond: B columns
      double* X = j < N ? M + j * SLD : B + (j - N) * SLD;
      if (i != k) X[i] = fma(-col[i], X[k], X[i]);
    }
    __syncthreads();
  }
  return true;
}

// The projected check for K <= 64 entirely in shared memory (buf: 6 * SMAT + 4 * SLD doubles):
// H^{-1}, A_hat = (I - H^{-1}) / gamma, F = exp(h A_hat) by Pade-13 scaling and squaring (Higham 2005),
// the chain z_q = F z_{q-1} in one warp, the residuals at every node.  Same outputs as hom_check.
__device__ static double hom_check_small(const ScanArgs& a, double* Zc, int K, double gam, double beta, double* buf,
                                         double* red, int* s_p) {
  const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                        1187353796428800.0,  129060195264000.0,   10559470521600.0,
                        670442572800.0,      33522128640.0,       1323241920.0,
                        40840800.0,          960960.0,            16380.0,
                        182.0,               1.0};
  const double theta13 = 5.371920351148152;
  const int ldh = a.kcap + 1;
  const int Np = (K + 3) & ~3;
  double *A1 = buf, *A2 = buf + SMAT, *A4 = buf + 2 * SMAT, *A6 = buf + 3 * SMAT, *T1 = buf + 4 * SMAT,
         *T2 = buf + 5 * SMAT;
  double* col = buf + 6 * SMAT;   // [SLD]
  double* hrow = col + SLD;       // last row of H^{-1}
  double* nrmc = hrow + SLD;      // column sums
  for (int t = threadIdx.x; t < 6 * SMAT; t += NT) buf[t] = 0.0;
  __syncthreads();
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int i = t % K, j = t / K;
    T1[i + j * SLD] = __ldcg(a.H + i + size_t(j) * ldh);
    if (i == j) T2[i + j * SLD] = 1.0;
  }
  __syncthreads();
  const double htail = __ldcg(a.H + K + size_t(K - 1) * ldh);
  if (!sm_gauss_jordan(K, T1, T2, K, col, s_p)) return INFINITY;  // T2 = H^{-1}
  for (int t = threadIdx.x; t < K; t += NT) hrow[t] = T2[(K - 1) + t * SLD];
  // A1 = h (I - H^{-1}) / gamma, its 1-norm, scaling
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int i = t % K, j = t / K;
    A1[i + j * SLD] = a.h * ((i == j ? 1.0 : 0.0) - T2[i + j * SLD]) / gam;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < K; j += NT) {
    double sum = 0.0;
    for (int i = 0; i < K; ++i) sum += fabs(A1[i + j * SLD]);
    nrmc[j] = sum;
  }
  __syncthreads();
  double nrm = 0.0;
  for (int j = 0; j < K; ++j) nrm = fmax(nrm, nrmc[j]);
  if (!isfinite(nrm)) return INFINITY;
  int sq = 0;
  if (nrm > theta13) sq = max(0, (int)ceil(log2(nrm / theta13)));
  if (sq > 0) {
    const double sc = ldexp(1.0, -sq);
    for (int t = threadIdx.x; t < K * K; t += NT) A1[(t % K) + (t / K) * SLD] *= sc;
    __syncthreads();
  }
  sm_gemm(Np, A1, A1, A2);
  sm_gemm(Np, A2, A2, A4);
  sm_gemm(Np, A4, A2, A6);
  // U = A1 [A6 (b13 A6 + b11 A4 + b9 A2) + b7 A6 + b5 A4 + b3 A2 + b1 I]
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int o = (t % K) + (t / K) * SLD;
    T1[o] = b[13] * A6[o] + b[11] * A4[o] + b[9] * A2[o];
  }
  __syncthreads();
  sm_gemm(Np, A6, T1, T2);
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int i = t % K, j = t / K, o = i + j * SLD;
    T2[o] += b[7] * A6[o] + b[5] * A4[o] + b[3] * A2[o] + (i == j ? b[1] : 0.0);
  }
  __syncthreads();
  sm_gemm(Np, A1, T2, T1);  // T1 = U
  // V = A6 (b12 A6 + b10 A4 + b8 A2) + b6 A6 + b4 A4 + b2 A2 + b0 I   (into A1: no longer needed)
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int o = (t % K) + (t / K) * SLD;
    T2[o] = b[12] * A6[o] + b[10] * A4[o] + b[8] * A2[o];
  }
  __syncthreads();
  sm_gemm(Np, A6, T2, A1);
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int i = t % K, j = t / K, o = i + j * SLD;
    const double v = A1[o] + b[6] * A6[o] + b[4] * A4[o] + b[2] * A2[o] + (i == j ? b[0] : 0.0);
    const double u = T1[o];
    T2[o] = v - u;   // (V - U) R = (V + U)
    T1[o] = v + u;
  }
  __syncthreads();
  if (!sm_gauss_jordan(K, T2, T1, K, col, s_p)) return INFINITY;  // T1 = R
  double *cur = T1, *nxt = T2;
  for (int t = threadIdx.x; t < SMAT; t += NT) nxt[t] = 0.0;  // T2 held the eliminated system
  __syncthreads();
  for (int q = 0; q < sq; ++q) {
    sm_gemm(Np, cur, cur, nxt);
    double* tmp = cur; cur = nxt; nxt = tmp;
  }
  // chain z_q = F z_{q-1} in ONE warp (lane l owns rows l and l + 32; z through shuffles)
  const double* F = cur;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int r0 = lane, r1 = lane + 32;
    double z0 = lane == 0 ? beta : 0.0, z1 = 0.0;
    if (r0 < K) Zc[r0] = z0;
    if (r1 < K) Zc[r1] = 0.0;
    for (int q = 1; q < a.s; ++q) {
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
      int j = 0;
      for (; j + 1 < K; j += 2) {
        const double zj = __shfl_sync(0xffffffffu, j < 32 ? z0 : z1, j & 31);
        const double zk = __shfl_sync(0xffffffffu, j + 1 < 32 ? z0 : z1, (j + 1) & 31);
        a0 = fma(F[r0 + j * SLD], zj, a0);
        a1 = fma(F[r1 + j * SLD], zj, a1);
        b0 = fma(F[r0 + (j + 1) * SLD], zk, b0);
        b1 = fma(F[r1 + (j + 1) * SLD], zk, b1);
      }
      if (j < K) {
        const double zj = __shfl_sync(0xffffffffu, j < 32 ? z0 : z1, j & 31);
        a0 = fma(F[r0 + j * SLD], zj, a0);
        a1 = fma(F[r1 + j * SLD], zj, a1);
      }
      z0 = r0 < K ? a0 + b0 : 0.0;
      z1 = r1 < K ? a1 + b1 : 0.0;
      if (r0 < K) Zc[size_t(q) * a.kcap + r0] = z0;
      if (r1 < K) Zc[size_t(q) * a.kcap + r1] = z1;
    }
  }
  __threadfence_block();
  __syncthreads();
  // residuals |h_{K+1,K} (H^{-1} z_q)_K| / gamma at every node (one warp per node)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double maxres = 0.0;
  for (int q = 1 + w; q < a.s; q += NT / 32) {
    double xp = 0.0;
    for (int r = lane; r < K; r += 32) xp = fma(hrow[r], Zc[size_t(q) * a.kcap + r], xp);
    xp = warp_sum(xp);
    maxres = fmax(maxres, fabs(htail * xp) / gam);
  }
  maxres = block_max(maxres, red);
  __syncthreads();
  return maxres;
}

// Projected check on the checker CTA: returns max_r residual; writes Zc[r][0..K).
__device__ static double hom_check(const ScanArgs& a, double* Zc, int K, double gam, double beta, double* z,
                                   double* zn, double* red, double* psm) {
  const int ld = a.kcap, ldh = a.kcap + 1;
  const size_t MM = size_t(ld) * ld;
  double* S0 = a.work;
  double* S1 = S0 + MM;
  double* S2 = S1 + MM;
  double* WK = S2 + MM;
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int i = t % K, j = t / K;
    S0[i + size_t(j) * ld] = __ldcg(a.H + i + size_t(j) * ldh);
  }
  __syncthreads();
  cta_identity(K, S1, ld, 1.0);
  cta_lu(K, S0, ld, a.iwork, red, kSolo, psm, HS_PSM);
  cta_lu_solve(K, S0, ld, a.iwork, S1, ld, K, kSolo, psm, HS_PSM, true);
  for (int t = threadIdx.x; t < K * K; t += NT) {
    const int i = t % K, j = t / K;
    S2[i + size_t(j) * ld] = a.h * ((i == j ? 1.0 : 0.0) - S1[i + size_t(j) * ld]) / gam;
  }
  __syncthreads();
  cta_expm_pade13(K, S2, ld, WK, ld, a.iwork, red, kSolo, psm, HS_PSM);
  const double htail = __ldcg(a.H + K + size_t(K - 1) * ldh);
  // chaining z_q = F z_{q-1} (F = e^{h A_hat}): F staged in shared memory when it fits, each row's
  // dot split over NT/K-way thread groups; the residuals |h_{K+1,K} (H^{-1} z_q)_K| / gamma are
  // evaluated afterwards from the stored z history (no block reduction inside the sequential loop)
  const bool fs = size_t(K) * K <= size_t(HS_PSM);
  double* F = fs ? psm : S2;
  const int ldf = fs ? K : ld;
  if (fs)
    for (int t = threadIdx.x; t < K * K; t += NT) F[t] = S2[(t % K) + size_t(t / K) * ld];
  for (int r = threadIdx.x; r < K; r += NT) z[r] = r == 0 ? beta : 0.0;
  __syncthreads();
  for (int r = threadIdx.x; r < K; r += NT) Zc[r] = z[r];
  const int ng = max(1, min(8, NT / max(K, 1)));  // thread groups per row
  const int jper = (K + ng - 1) / ng;
  if (fs && K <= 64) {
    // small spaces (the usual case): the whole chain in ONE warp, no block barriers -- lane l owns rows
    // l and l + 32 of the state, the products read F from shared memory and z through shuffles
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const int r0 = lane, r1 = lane + 32;
      double z0 = lane == 0 ? beta : 0.0, z1 = 0.0;
      const double* F0 = F + (r0 < K ? r0 : 0);
      const double* F1 = F + (r1 < K ? r1 : 0);
      for (int q = 1; q < a.s; ++q) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        int j = 0;
        for (; j + 1 < K; j += 2) {
          const double zj = __shfl_sync(0xffffffffu, j < 32 ? z0 : z1, j & 31);
          const double zk = __shfl_sync(0xffffffffu, j + 1 < 32 ? z0 : z1, (j + 1) & 31);
          a0 = fma(F0[size_t(j) * K], zj, a0);
          a1 = fma(F1[size_t(j) * K], zj, a1);
          b0 = fma(F0[size_t(j + 1) * K], zk, b0);
          b1 = fma(F1[size_t(j + 1) * K], zk, b1);
        }
        if (j < K) {
          const double zj = __shfl_sync(0xffffffffu, j < 32 ? z0 : z1, j & 31);
          a0 = fma(F0[size_t(j) * K], zj, a0);
          a1 = fma(F1[size_t(j) * K], zj, a1);
        }
        z0 = r0 < K ? a0 + b0 : 0.0;
        z1 = r1 < K ? a1 + b1 : 0.0;
        if (r0 < K) Zc[size_t(q) * a.kcap + r0] = z0;
        if (r1 < K) Zc[size_t(q) * a.kcap + r1] = z1;
      }
    }
    __threadfence_block();
    __syncthreads();
  } else
  for (int q = 1; q < a.s; ++q) {
    const int r = threadIdx.x % K, gq = threadIdx.x / K;
    if (threadIdx.x < ng * K) {
      const int j0 = gq * jper, j1 = min(K, j0 + jper);
      double v0 = 0.0, v1 = 0.0;
      int j = j0;
      for (; j + 1 < j1; j += 2) {
        v0 = fma(F[r + size_t(j) * ldf], z[j], v0);
        v1 = fma(F[r + size_t(j + 1) * ldf], z[j + 1], v1);
      }
      if (j < j1) v0 = fma(F[r + size_t(j) * ldf], z[j], v0);
      zn[gq * K + r] = v0 + v1;
    }
    __syncthreads();
    for (int rr = threadIdx.x; rr < K; rr += NT) {
      double v = 0.0;
      for (int g2 = 0; g2 < ng; ++g2) v += zn[g2 * K + rr];
      z[rr] = v;
      Zc[size_t(q) * a.kcap + rr] = v;
    }
    __syncthreads();
  }
  // residuals of all nodes in parallel (one warp per node)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double maxres = 0.0;
  for (int q = 1 + w; q < a.s; q += NT / 32) {
    double xp = 0.0;
    for (int r = lane; r < K; r += 32) xp = fma(S1[(K - 1) + size_t(r) * ld], __ldcg(Zc + size_t(q) * a.kcap + r), xp);
    xp = warp_sum(xp);
    maxres = fmax(maxres, fabs(htail * xp) / gam);
  }
  maxres = block_max(maxres, red);
  __syncthreads();
  return maxres;
}

__global__ void __launch_bounds__(NT, 1) k_hom_scan(ScanArgs a) {
  __shared__ double red[32];
  __shared__ Aff wsm[NT / 32 + 1];
  __shared__ int s_dec, s_dec2;
  extern __shared__ double dyn[];  // hv, hv2: KSMALL_MAX + 8 each; xs: NT * RPT_MAX; LU scratch HS_PSM
  double* hv = dyn;
  double* hv2 = dyn + KSMALL_MAX + 8;
  double* xs = hv2 + KSMALL_MAX + 8;
  double* xg = xs + NT * RPT_MAX;     // workers: gathered exchange-1 rows [nw][8]; checker: LU scratch from here
  double* Vs = xg + XG_DOUBLES;       // workers: the CTA's rows of the first vcap basis columns
  __shared__ Aff3 wsm3[NT / 32 + 1];
  const int c = blockIdx.x;
  const bool checker = c == a.nw;
  const int n = a.n, s = a.s, rpt = a.rpt;
  const int pw = a.kcap + 8;       // partial row width: [0, kcap] dots, +1 norm, +2 SM dot, +3 beta
  const int PN = a.kcap + 1, PF = a.kcap + 2, PBETA = a.kcap + 3;
  unsigned* bar = a.bar;
  int* fl = a.flags;
  // own rows: g = row0 + threadIdx.x * rpt + q
  const int row0 = c * a.seg;
  const int rend = min(n, row0 + a.seg);
  double uh[RPT_MAX], xr[RPT_MAX], vr[RPT_MAX];
  int kconv_prev = 0;  // checker: converged dimension of the previous subinterval (thread 0)
  Xch X;
  X.base = a.xch; X.nw = a.nw; X.pw = a.kcap + 8; X.c = c;

  // ---- subinterval 0: no homogeneous part; u_hat(T_1) = Y(T_1) (its waveform u0 + Y is written by
  // k_scan_output after the scan)
  if (!checker) {
    double b2 = 0.0;
    _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
      const int g = row0 + threadIdx.x * rpt + q;
      uh[q] = 0.0;
      if (g >= rend) continue;
      uh[q] = a.Y[size_t(s - 1) * n + g];
      b2 = fma(uh[q], uh[q], b2);
    }
    b2 = block_sum(b2, red);
    if (threadIdx.x == 0) a.partA[size_t(c) * pw + PBETA] = b2;
    if (c == 0 && threadIdx.x == 0) {
      a.kc[0] = 0;
      a.koff[0] = 0;
      a.koff[1] = 0;
    }
  }
  gbar(bar + B_ACNT, bar + B_AGEN, a.nw + 1);

  for (int i = 1; i < a.P; ++i) {
    grid_reduce(a.partA, pw, a.nw, PBETA, 1, hv);
    const double beta = sqrt(hv[0]);
    const double gam = a.gam[i];
    const size_t fo = size_t(i) * n;
    // this subinterval's basis: archived in the pool when it still has room for a full space
    const int koff = __ldcg(a.koff + i);
    const bool arch = koff >= 0 && koff + a.kcap + 1 <= a.pool_cols;
    double* Vi = arch ? a.Vpool + size_t(koff) * n : a.V;
    double* Zi = a.Zc + size_t(i) * a.s * a.kcap;
    gbar(bar + B_ACNT, bar + B_AGEN, a.nw + 1);  // everyone has read beta before partA is reused
    if (checker) {
      // ---------------------------------------------------------------- checker CTA
      if (beta > 0.0) {
        const double crit = a.eta * beta / ((s - 1) * a.h);
        double* z = hv;
        double* zn = hv2;
        // first check just below the previous subinterval's converged dimension (the operators of
        // neighbouring subintervals are close), then extrapolate the residual decay
        int target = min(max(4, kconv_prev - 2), a.kcap - 1), Kprev = -1;
        double qprev = -1.0;
        while (true) {
          if (threadIdx.x == 0) {
            int K;
            while (true) {
              K = vload(fl + F_STEPS);
              const int bk = vload(fl + F_BREAK);
              if (bk > 0) { K = bk; break; }
              if (K >= target) break;
              __nanosleep(64);
            }
            __threadfence();
            s_dec = K;
          }
          __syncthreads();
          const int K = s_dec;
          const bool brk = vload(fl + F_BREAK) == K;
          const long long tc0 = clock64();
          const double res = K <= SLD ? hom_check_small(a, Zi, K, gam, beta, dyn, red, &s_dec2)
                                      : hom_check(a, Zi, K, gam, beta, z, zn, red, xs + NT * RPT_MAX);
          if (threadIdx.x == 0) {
            fl[F_NCHECK] += 1;
            fl[F_CHKCYC] += int((clock64() - tc0) >> 10);
            int result = 0;
            if (brk || res <= crit) {
              result = K;
              kconv_prev = K;
            }
            else if (K >= a.kcap - 1) result = -1;
            if (result != 0) {
              __threadfence();
              atomicExch(fl + F_RESULT, result);
              atomicMax(fl + F_KMAX, K);
            } else {
              const double qv = res / crit;
              int nt = K + 2;
              if (Kprev >= 0 && qprev > 0.0 && qv > 0.0 && qv < qprev) {
                const double slope = (log(qv) - log(qprev)) / double(K - Kprev);
                nt = (int)ceil(K + log(0.5 / qv) / slope);
              }
              target = min(max(nt, K + 1), min(2 * K, a.kcap - 1));
              Kprev = K;
              qprev = qv;
            }
            s_dec = result;
          }
          __syncthreads();
          if (s_dec != 0) break;
        }
      }
    } else {
      // ---------------------------------------------------------------- workers
      const double inv = beta > 0.0 ? 1.0 / beta : 0.0;
      // this subinterval's factor rows of the CTA's segment, in registers for all Arnoldi steps
      double f_l[RPT_MAX], f_di[RPT_MAX], f_a[RPT_MAX], f_z[RPT_MAX], f_w[RPT_MAX];
      _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
        const int g = row0 + threadIdx.x * rpt + q;
        const bool ok = g < rend;
        f_l[q] = ok ? a.fl[fo + g] : 0.0;
        f_di[q] = ok ? a.fdinv[fo + g] : 0.0;
        f_a[q] = ok ? -f_di[q] * a.fsup[fo + g] : 1.0;
        f_z[q] = ok && a.periodic ? a.fz[fo + g] : 0.0;
        f_w[q] = ok && a.periodic ? a.fw[fo + g] : 0.0;
        vr[q] = uh[q] * inv;
        if (ok) {
          if (0 < a.vcap) Vs[threadIdx.x * rpt + q] = vr[q];
          else Vi[g] = vr[q];
        }
      }
      __syncthreads();
      int Kc = 0;     // converged dimension (0: beta == 0, no homogeneous part)
      int kused = 0;  // basis columns written (Arnoldi steps performed + 1)
      if (beta > 0.0) {
        for (int k = 0;; ++k) {
          kused = k + 1;
          // A: y_g = -l_g y_{g-1} + b_g over own rows as y_g = ya_g cy + yb_g (cy: carry from the lower
          // segments); x_g = a_g x_{g+1} + di_g y_g composed over own rows with the offset affine in cy
          int dec_pref = 0;
          if (c == 0 && threadIdx.x == 0) dec_pref = vload(fl + F_RESULT);  // in flight during the scans
          Aff m{1.0, 0.0};
          double fdot = 0.0;
          _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
            const int g = row0 + threadIdx.x * rpt + q;
            if (g < rend) {
              m = after(m, Aff{-f_l[q], vr[q]});
              fdot = fma(f_w[q], vr[q], fdot);
            }
          }
          Aff tot;
          const Aff pre = block_excl_scan<false>(m, threadIdx.x, wsm, tot);
          double ya[RPT_MAX], yb[RPT_MAX];
          {
            double al = pre.A, be = pre.B;
            _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
              const int g = row0 + threadIdx.x * rpt + q;
              if (g < rend) {
                al = -f_l[q] * al;
                be = fma(-f_l[q], be, vr[q]);
              }
              ya[q] = al;
              yb[q] = be;
            }
          }
          Aff3 mb{1.0, 0.0, 0.0};
          _Pragma("unroll") for (int q = RPT_MAX - 1; q >= 0; --q) if (q < rpt) {
            const int g = row0 + threadIdx.x * rpt + q;
            if (g < rend) mb = after3(mb, Aff3{f_a[q], f_di[q] * yb[q], f_di[q] * ya[q]});
          }
          Aff3 totb;
          const Aff3 preb = block_excl_scan3_rev(mb, NT - 1 - threadIdx.x, wsm3, totb);
          if (a.periodic) fdot = block_sum(fdot, red);
          if (threadIdx.x == 0) {
            double d = 0.0;
            if (c == 0) {  // leader: decision for this step
              int dd = dec_pref;
              if (dd == 0 && (k >= a.kcap - 1 || vload(fl + F_BREAK) > 0)) {  // no room / invariant space
                while ((dd = vload(fl + F_RESULT)) == 0) __nanosleep(64);
              }
              d = double(dd);
            }
            xs[0] = tot.A; xs[1] = tot.B; xs[2] = totb.A; xs[3] = totb.B0; xs[4] = totb.B1; xs[5] = fdot;
            xs[6] = d; xs[7] = 0.0;
          }
          __syncthreads();
          xch_publish(X, xs, 8);
          xch_gather(X, 8, xg);
          const int dec = int(xg[6]);
          if (dec != 0) {
            Kc = dec;
            break;
          }
          // B: all segments' maps composed by warp 0 (every CTA identically): own carries and the SM dot
          if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            const int per = (a.nw + 31) / 32;
            // forward: cy at the start of each of the lane's segments
            Aff run{1.0, 0.0};
            for (int u = 0; u < per; ++u) {
              const int cc = lane * per + u;
              if (cc < a.nw) run = after(run, Aff{xg[cc * 8 + 0], xg[cc * 8 + 1]});
            }
            Aff inc = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double pa = __shfl_up_sync(0xffffffffu, inc.A, o), pb = __shfl_up_sync(0xffffffffu, inc.B, o);
              if (lane >= o) inc = after(Aff{pa, pb}, inc);
            }
            double cyl = __shfl_up_sync(0xffffffffu, inc.B, 1);  // carry into the lane's first segment
            if (lane == 0) cyl = 0.0;
            // backward maps x_first = A x_in + (B0 + B1 cy) of the lane's segments, composed descending
            Aff runb{1.0, 0.0};
            double cys[8];
            {
              double cyv = cyl;
              for (int u = 0; u < per; ++u) {
                const int cc = lane * per + u;
                cys[u] = cyv;
                if (cc < a.nw) cyv = fma(xg[cc * 8 + 0], cyv, xg[cc * 8 + 1]);
              }
            }
            for (int u = per - 1; u >= 0; --u) {
              const int cc = lane * per + u;
              if (cc < a.nw) runb = after(runb, Aff{xg[cc * 8 + 2], fma(xg[cc * 8 + 4], cys[u], xg[cc * 8 + 3])});
            }
            Aff incb = runb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const double pa = __shfl_down_sync(0xffffffffu, incb.A, o), pb = __shfl_down_sync(0xffffffffu, incb.B, o);
              if (lane + o < 32) incb = after(Aff{pa, pb}, incb);
            }
            double cxl = __shfl_down_sync(0xffffffffu, incb.B, 1);  // x entering the lane's LAST segment from above
            if (lane == 31) cxl = 0.0;
            // own segment: walk down from the lane's last segment to c
            const int lo = c / per;
            if (lane == lo) {
              double cxv = cxl;
              for (int u = per - 1; u > c - lo * per; --u) {
                const int cc = lane * per + u;
                if (cc < a.nw) cxv = fma(xg[cc * 8 + 2], cxv, fma(xg[cc * 8 + 4], cys[u], xg[cc * 8 + 3]));
              }
              hv[0] = cys[c - lo * per];
              hv[1] = cxv;
            }
            double fs = 0.0;
            for (int u = 0; u < per; ++u) {
              const int cc = lane * per + u;
              if (cc < a.nw) fs += xg[cc * 8 + 5];
            }
            fs = warp_sum(fs);
            if (lane == 0) hv[2] = fs;
          }
          __syncthreads();
          const double cy = hv[0], cx = hv[1], fsm = a.periodic ? hv[2] : 0.0;
          {
            double x = fma(preb.A, cx, fma(preb.B1, cy, preb.B0));
            _Pragma("unroll") for (int q = RPT_MAX - 1; q >= 0; --q) if (q < rpt) {
              const int g = row0 + threadIdx.x * rpt + q;
              if (g < rend) {
                const double y = fma(ya[q], cy, yb[q]);
                x = fma(f_a[q], x, f_di[q] * y);
                xr[q] = fma(-fsm, f_z[q], x);
              }
            }
          }
          __syncthreads();  // hv free again
          const int kk = k + 1;  // columns 0..k
          seg_dots2(Vs, a.segp, a.vcap, Vi, n, row0, rend - row0, kk, xr, rpt, xs, hv2);
          xch_publish(X, hv2, kk + 1);
          // C: h = V^T x; x -= V h; pass-2 dots
          xch_reduce(X, kk + 1, hv);  // h = V^T x and ||x||^2 (at kk)
          const double nrm0 = sqrt(hv[kk]);
          _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
            const int g = row0 + threadIdx.x * rpt + q;
            if (g < rend) {
              const int l = threadIdx.x * rpt + q;
              double v0 = xr[q], v1 = 0.0;
              const int ks = min(kk, a.vcap);
              int j = 0;
              for (; j + 1 < ks; j += 2) {
                v0 = fma(-hv[j], Vs[size_t(j) * a.segp + l], v0);
                v1 = fma(-hv[j + 1], Vs[size_t(j + 1) * a.segp + l], v1);
              }
              if (j < ks) v0 = fma(-hv[j], Vs[size_t(j) * a.segp + l], v0);
              for (j = ks; j < kk; ++j) v0 = fma(-hv[j], Vi[size_t(j) * n + g], v0);
              xr[q] = v0 + v1;
            }
          }
          seg_dots2(Vs, a.segp, a.vcap, Vi, n, row0, rend - row0, kk, xr, rpt, xs, hv2);
          xch_publish(X, hv2, kk + 1);
          // D: second pass, norm, new column
          xch_reduce(X, kk + 1, hv2);
          double h2n = 0.0;
          for (int j = 0; j < kk; ++j) h2n = fma(hv2[j], hv2[j], h2n);
          const double hn = sqrt(fmax(hv2[kk] - h2n, 0.0));
          const bool brk = !(hn > a.defl * nrm0);
          const double sc = brk ? 0.0 : 1.0 / hn;
          _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
            const int g = row0 + threadIdx.x * rpt + q;
            if (g < rend) {
              const int l = threadIdx.x * rpt + q;
              double v0 = xr[q], v1 = 0.0;
              const int ks = min(kk, a.vcap);
              int j = 0;
              for (; j + 1 < ks; j += 2) {
                v0 = fma(-hv2[j], Vs[size_t(j) * a.segp + l], v0);
                v1 = fma(-hv2[j + 1], Vs[size_t(j + 1) * a.segp + l], v1);
              }
              if (j < ks) v0 = fma(-hv2[j], Vs[size_t(j) * a.segp + l], v0);
              for (j = ks; j < kk; ++j) v0 = fma(-hv2[j], Vi[size_t(j) * n + g], v0);
              vr[q] = (v0 + v1) * sc;
              // columns resident in shared memory reach the global archive once, after the loop (no
              // global stores in flight when the exchange's fence runs)
              if (kk < a.vcap) Vs[size_t(kk) * a.segp + l] = vr[q];
              else Vi[size_t(kk) * n + g] = vr[q];
            }
          }
          if (c == 0) {
            const int ldh = a.kcap + 1;
            for (int j = threadIdx.x; j <= kk; j += NT)
              a.H[j + size_t(k) * ldh] = j < kk ? hv[j] + hv2[j] : (brk ? 0.0 : hn);
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
              if (brk) atomicCAS(fl + F_BREAK, 0, kk);
              atomicExch(fl + F_STEPS, kk);
            }
          }
          __syncthreads();  // hv, hv2, Vs column kk complete before the next step reads them
        }
      }
      if (Kc < 0) {
        if (c == 0 && threadIdx.x == 0) atomicExch(fl + F_ERR, 1);
        Kc = 0;
      }
      // the shared-memory columns of this subinterval's basis -> global (archive for k_scan_output /
      // the in-scan waveform update below); every thread stores the rows it reads back later
      {
        const int nc = min(max(Kc, 0), a.vcap);
        _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
          const int g = row0 + threadIdx.x * rpt + q;
          if (g < rend) {
            const int l = threadIdx.x * rpt + q;
            for (int j = 0; j < nc; ++j) Vi[size_t(j) * n + g] = Vs[size_t(j) * a.segp + l];
          }
        }
      }
      // archived: only the end value u_hat(T_i) = Y(T_i) + V z(T_i) here (the waveform at all nodes is
      // written by k_scan_output after the scan); otherwise the full waveform update in place
      const size_t yo = size_t(i) * s * n;
      double b2 = 0.0;
      if (arch) {
        for (int t = threadIdx.x; t < Kc; t += NT) hv[t] = __ldcg(Zi + size_t(s - 1) * a.kcap + t);
        __syncthreads();
        _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
          const int g = row0 + threadIdx.x * rpt + q;
          uh[q] = 0.0;
          if (g >= rend) continue;
          double w = 0.0;
          for (int j = 0; j < Kc; ++j) w = fma(Vi[size_t(j) * n + g], hv[j], w);
          uh[q] = a.Y[yo + size_t(s - 1) * n + g] + w;
          b2 = fma(uh[q], uh[q], b2);
        }
        b2 = block_sum(b2, red);
      } else {
        for (int t = threadIdx.x; t < s * Kc && Kc > 0 && s * Kc <= KSMALL_MAX; t += NT)
          hv[t] = __ldcg(Zi + size_t(t / Kc) * a.kcap + t % Kc);
        __syncthreads();
        double mx = 0.0;
        _Pragma("unroll") for (int q = 0; q < RPT_MAX; ++q) if (q < rpt) {
          const int g = row0 + threadIdx.x * rpt + q;
          uh[q] = 0.0;
          if (g >= rend) continue;
          for (int r = 0; r < s; ++r) {
            double w = 0.0;
            if (s * Kc <= KSMALL_MAX) {
              for (int j = 0; j < Kc; ++j) w = fma(Vi[size_t(j) * n + g], hv[r * Kc + j], w);
            } else {
              for (int j = 0; j < Kc; ++j) w = fma(Vi[size_t(j) * n + g], __ldcg(Zi + size_t(r) * a.kcap + j), w);
            }
            const size_t kx = yo + size_t(r) * n + g;
            const double uhr = a.Y[kx] + w;
            const double un = a.u0[g] + uhr;
            mx = fmax(mx, fabs(un - a.Uold[kx]));
            if (!isfinite(un)) mx = INFINITY;
            a.Unew[kx] = un;
            if (r == s - 1) uh[q] = uhr;
          }
          b2 = fma(uh[q], uh[q], b2);
        }
        mx = block_max(mx, red);
        b2 = block_sum(b2, red);
        if (threadIdx.x == 0) atomic_max_nonneg(a.delta, mx);
      }
      if (threadIdx.x == 0) a.partA[size_t(c) * pw + PBETA] = b2;
      if (c == 0 && threadIdx.x == 0) {
        fl[F_NSTEPS] += kused;
        a.kc[i] = arch ? Kc : -1;
        if (i + 1 < a.P) a.koff[i + 1] = arch ? koff + kused + 1 : koff;
      }
    }
    // reset the per-subinterval flags (nobody reads them until after the barrier)
    if (c == 0 && threadIdx.x == 0) {
      fl[F_STEPS] = 0;
      fl[F_RESULT] = 0;
      fl[F_DECISION] = 0;
      fl[F_BREAK] = 0;
      __threadfence();
    }
    gbar(bar + B_ACNT, bar + B_AGEN, a.nw + 1);
    if (vload(fl + F_ERR)) return;
  }
}

// The waveform update of every archived subinterval, after the scan (all subintervals in parallel):
//   u_{k+1}(t_{i,r}) = u0 + Y_i(t_r) + V_i z_i(t_r),  delta = max |u_{k+1} - u_k|    (Eq.(updateSolution))
// One thread per row; the node coefficients z_i(t_r) staged in shared memory 32 columns at a time.
constexpr int OUT_SMAX = 64;
constexpr int OUT_SG = 32;  // nodes per CTA (blockIdx.z selects the node group: 64 registers of accumulators)
__global__ void __launch_bounds__(NT, 2) k_scan_output(int s, int n, int kcap, const double* u0, const double* Y,
                                                       const double* Uold, double* Unew, const double* Vpool,
                                                       const int* koff, const int* kc, const double* Zc,
                                                       double* delta) {
  const int i = blockIdx.y;
  const int K = kc[i];
  if (K < 0) return;  // this subinterval's waveform was written inside the scan
  const int rb = blockIdx.z * OUT_SG;       // first node of this CTA's group
  const int ns = min(OUT_SG, s - rb);
  if (ns <= 0) return;
  __shared__ double Zs[OUT_SG][33];
  __shared__ double red[32];
  const int g = blockIdx.x * NT + threadIdx.x;
  double acc[OUT_SG];
#pragma unroll
  for (int r = 0; r < OUT_SG; ++r) acc[r] = 0.0;
  const double* V = Vpool + size_t(koff[i]) * n;
  const double* Z = Zc + size_t(i) * s * kcap;
  for (int j0 = 0; j0 < K; j0 += 32) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < OUT_SG * 32; idx += NT) {
      const int r = idx / 32, jj = idx % 32;
      Zs[r][jj] = (r < ns && j0 + jj < K) ? __ldcg(Z + size_t(rb + r) * kcap + j0 + jj) : 0.0;
    }
    __syncthreads();
    if (g < n) {
      const int jn = min(32, K - j0);
      for (int jj = 0; jj < jn; jj += 4) {  // four basis columns per round: independent loads in flight
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = jj + u < jn ? V[size_t(j0 + jj + u) * n + g] : 0.0;
#pragma unroll
        for (int r = 0; r < OUT_SG; ++r) {
          double a = acc[r];
#pragma unroll
          for (int u = 0; u < 4; ++u) a = fma(v[u], Zs[r][jj + u], a);   // Zs is zero beyond K
          acc[r] = a;
        }
      }
    }
  }
  double mx = 0.0;
  if (g < n) {
    const double ug = u0[g];
#pragma unroll
    for (int r0 = 0; r0 < OUT_SG; r0 += 8) {  // eight nodes per round: 16 independent loads in flight
      double yv[8], uo[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const size_t k = (size_t(i) * s + rb + r0 + u) * n + g;
        yv[u] = r0 + u < ns ? Y[k] : 0.0;
        uo[u] = r0 + u < ns ? Uold[k] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (r0 + u < ns) {
          const size_t k = (size_t(i) * s + rb + r0 + u) * n + g;
          const double un = ug + yv[u] + acc[r0 + u];
          mx = fmax(mx, fabs(un - uo[u]));
          if (!isfinite(un)) mx = INFINITY;
          Unew[k] = un;
        }
    }
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) atomic_max_nonneg(delta, mx);
}

// worker CTAs of the scan: one per 256 rows (at most 147)
static int scan_workers(int n) { return std::min(147, cdiv(n, NT)); }

bool hom_scan_ok(int n, int kcap) { return kcap <= KSMALL_MAX && n <= 147 * NT * RPT_MAX; }

// archive of the scan's bases (outputs after the scan): on average 96 columns per subinterval;
// subintervals beyond it write their waveform inside the scan
static long long scan_pool_cols(int P, int kcap) { return (long long)P * std::min(kcap + 1, 96) + kcap + 1; }

size_t hom_scan_bytes(int n, int s, int kcap, int P) {
  const int nw = scan_workers(n);
  const size_t pw = kcap + 8;
  return sizeof(double) * (size_t(kcap + 1) * n + size_t(kcap + 1) * kcap + size_t(P) * s * kcap + 5 * nw * pw +
                           4 * nw + 10 * size_t(kcap) * kcap + size_t(scan_pool_cols(P, kcap)) * n) +
         sizeof(int) * (kcap + F_NFLAGS + 2 * P) + 4 * sizeof(unsigned) + 20 * 256;  // + arena alignment
}

int launch_hom_scan(cudaStream_t st, const Factors& F, const double* gam, int P, int s, int n, int kcap, double h,
                    double eta, double defl, const double* u0, const double* Y, const double* Uold, double* Unew,
                    double* delta, char* ws, size_t ws_bytes, int* kscan_rec, double* diag) {
  Arena ar{ws, ws_bytes, 0};
  ScanArgs a{};
  a.P = P; a.s = s; a.n = n; a.kcap = kcap; a.periodic = F.periodic;
  a.nw = scan_workers(n);
  a.seg = cdiv(n, a.nw);
  a.rpt = cdiv(a.seg, NT);
  if (a.rpt > RPT_MAX) fail(1, "hom_scan: n too large for the persistent scan");
  a.fl = F.l; a.fdinv = F.dinv; a.fsup = F.sup; a.fz = F.z; a.fw = F.w;
  a.gam = gam; a.h = h; a.eta = eta; a.defl = defl;
  a.u0 = u0; a.Y = Y; a.Uold = Uold; a.Unew = Unew; a.delta = delta;
  const size_t pw = kcap + 8;
  a.V = ar.take<double>(size_t(kcap + 1) * n);
  a.H = ar.take<double>(size_t(kcap + 1) * kcap);
  a.Zc = ar.take<double>(size_t(P) * s * kcap);
  a.pool_cols = scan_pool_cols(P, kcap);
  a.Vpool = ar.take<double>(size_t(a.pool_cols) * n);
  a.koff = ar.take<int>(P);
  a.kc = ar.take<int>(P);
  if (s > OUT_SMAX) fail(1, "hom_scan: s > 64");
  a.partA = ar.take<double>(a.nw * pw);
  a.partB = ar.take<double>(a.nw * pw);
  a.maps = ar.take<double>(4 * a.nw);
  a.xch = ar.take<double>(3 * size_t(a.nw) * pw);
  a.segp = a.seg;
  a.vcap = std::min(VS_DOUBLES / a.segp, kcap + 1);
  a.work = ar.take<double>(10 * size_t(kcap) * kcap);
  a.iwork = ar.take<int>(kcap);
  a.flags = ar.take<int>(F_NFLAGS);
  a.bar = ar.take<unsigned>(4);
  if (ar.off > ws_bytes) fail(2, "hom_scan workspace too small");
  PEXP_CUDA_TRY(cudaMemsetAsync(a.flags, 0, F_NFLAGS * sizeof(int), st));
  PEXP_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 4 * sizeof(unsigned), st));
  PEXP_CUDA_TRY(cudaMemsetAsync(a.xch, 0xFF, 3 * size_t(a.nw) * pw * sizeof(double), st));  // sentinel
  PEXP_CUDA_TRY(cudaMemsetAsync(a.H, 0, size_t(kcap + 1) * kcap * sizeof(double), st));
  {
    // algorithmic bytes: the waveform pass (Y, Uold read; Unew write) per subinterval
    ProfScope ps(PC_SCAN, st, 0.0, 0.0);  // latency-bound chain
    void* args[] = {&a};
    const size_t smem = sizeof(double) * SCAN_SMEM_DOUBLES;
    PEXP_CUDA_TRY(cudaFuncSetAttribute(k_hom_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PEXP_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_hom_scan, dim3(a.nw + 1), dim3(NT), args, smem, st));
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
  {
    // algorithmic: Y, u_k read, u_{k+1} written at every node; the archived bases read once (~32 columns)
    ProfScope ps(PC_SCANOUT, st, double(P) * s * n * 24.0 + double(P) * 32.0 * n * 8.0, 2.0 * double(P) * s * n * 32.0);
    k_scan_output<<<dim3(cdiv(n, NT), P, cdiv(s, OUT_SG)), NT, 0, st>>>(s, n, kcap, u0, Y, Uold, Unew, a.Vpool, a.koff, a.kc, a.Zc,
                                                       delta);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
  int hf[F_NFLAGS];
  PEXP_CUDA_TRY(cudaMemcpyAsync(hf, a.flags, sizeof(hf), cudaMemcpyDeviceToHost, st));
  host_sync(st);
  if (hf[F_ERR]) fail(4 /* PEXP_ENOCONV */, "Krylov capacity reached (homogeneous scan)");
  if (kscan_rec) PEXP_CUDA_TRY(cudaMemcpy(kscan_rec, a.kc, P * sizeof(int), cudaMemcpyDeviceToHost));
  if (diag) {
    diag[0] += hf[F_NSTEPS];
    diag[1] += hf[F_NCHECK];
    diag[2] += double(hf[F_CHKCYC]) * 1024.0;
  }
  return hf[F_KMAX];
}

}  // namespace pexp
