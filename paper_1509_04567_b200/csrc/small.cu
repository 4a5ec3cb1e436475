// small.cu — one-CTA-per-evaluation dense kernels on the small projected quantities:
//   * k_sym_eig_select  : cyclic parallel Jacobi eigensolver of an s x s source Gram matrix
//                         (subsystem 3, "Gram matrix plus small Jacobi eigensolve") and the
//                         pass selection of the two-pass rank-revealing source SVD
//   * k_block_chol      : scaled, deflating Cholesky of a block Gram matrix -> R, R^{-1}
//                         (Cholesky-QR of Arnoldi blocks and of the source basis)
//   * k_onesided_svd    : one-sided (Hestenes) Jacobi SVD of the projected coefficient matrix
//                         C = U^T G, final truncation m_j = #{sigma > tau*sigma_1}
//   * k_build_final     : selection matrices for U_final = U Q[:, :m] and coefficient rows
//   * k_spline          : not-a-knot cubic p(t) per coefficient row
//   * k_small_problem   : projected SaI problem: H^{-1}, A_hat = (I - H^{-1})/gamma, Pade-13
//                         exponential of the augmented matrix, exact chaining over the cubic
//                         pieces, residual norms at every node (subsystem 4)
#include <cooperative_groups.h>
#include <cstdlib>
#include "common.cuh"
#include "dense.cuh"
#include "kernels.cuh"

namespace pexp {

constexpr int MAXS = 64;
namespace cg = cooperative_groups;
// k_small_problem dynamic shared memory: replicated state 2*KSMALL_MAX, row partials CH_PSUM,
// own rows KSMALL_MAX, residual partials of every piece RING_N*MAXS, then the CTA's slice of F
// (FS_CAP doubles)
constexpr int CH_PSUM = KSMALL_MAX + 32;
#if PEXP_GEMM_TM >= 128
constexpr size_t SP_DYN = 180 * 1024;
constexpr size_t HOM_DYN = 160 * 1024;
constexpr int SMALL_MINB = 1;
#else
constexpr size_t SP_DYN = 72 * 1024;   // two CTAs per SM (with ~23 KB static shared memory)
constexpr size_t HOM_DYN = 72 * 1024;
constexpr int SMALL_MINB = 2;
#endif
constexpr size_t HOM_FS_CAP = HOM_DYN / 8 - 2 * 256;
constexpr int RING_N = 64;  // pieces whose residual partials are kept (s - 1 <= 63)
constexpr size_t FS_CAP = SP_DYN / 8 - (2 * KSMALL_MAX + CH_PSUM + KSMALL_MAX + RING_N * MAXS);
constexpr size_t SM2 = 2 * MAXS * (MAXS + 1) * sizeof(double);  // two padded 64x64 tiles

// Cluster size so that (evaluations x cluster) fills the 148 SMs (portable maximum 8).
static int cluster_size_for(int E) {
  int cs = 1;
  while (cs < 8 && E * cs * 2 <= 148 * SMALL_MINB) cs *= 2;
  // (16-CTA clusters measured slower here: E=8, N=208 expm 1.80 ms vs 1.15 ms with 8)
  return cs;
}

template <class Kern, class... Args>
static void launch_clustered(Kern kern, int nclusters, int cs, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nclusters * cs);
  cfg.blockDim = dim3(PEXP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PEXP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
}

__device__ inline void jacobi_pair(int Ne, int r, int k, int& p, int& q) {
  if (k == 0) {
    p = r;
    q = Ne - 1;
  } else {
    p = (r + k) % (Ne - 1);
    q = (r - k + (Ne - 1)) % (Ne - 1);
  }
  if (p > q) { int t = p; p = q; q = t; }
}

__device__ inline void sym_schur2(double app, double aqq, double apq, double& c, double& s) {
  if (fabs(apq) < 1e-300) { c = 1.0; s = 0.0; return; }
  double tau = (aqq - app) / (2.0 * apq);
  double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + hypot(1.0, tau));
  c = 1.0 / sqrt(1.0 + t * t);
  s = t * c;
}

// ---------------------------------------------------------------- Jacobi eig + selection
// G: [E][s][s] (col-major s x s).  Pass `pass` of the two-pass SVD: keep eigenpairs with
// sigma_i = sqrt(lambda_i) > theta*sigma_max(pass) and > 0.5*tau*sigma1 (sigma1 from pass 0),
// write Msel[:, off + c] = q_i / sigma_i (all other columns 0), off += kept.
// Parallel cyclic Jacobi (round-robin pairing): per round the Ne/2 disjoint rotations are
// computed by Ne/2 threads, then every thread applies both rotations to ONE 2x2 block
// (rows {p_k,q_k} x columns {p_l,q_l}) of A and one column pair of Q — two barriers per round.
constexpr int EIG_THREADS = 1024;
__global__ void __launch_bounds__(EIG_THREADS)
k_sym_eig_select(int s, const double* G, double* lam_out, double* Msel, int* off, double* sigma1,
                 int pass, double tau, double theta, const int* active) {
  const int e = blockIdx.x;
  extern __shared__ double dsm[];
  double (*A)[MAXS + 1] = reinterpret_cast<double (*)[MAXS + 1]>(dsm);
  double (*Q)[MAXS + 1] = reinterpret_cast<double (*)[MAXS + 1]>(dsm + MAXS * (MAXS + 1));
  __shared__ double rc[MAXS / 2], rs[MAXS / 2];
  __shared__ int rp[MAXS / 2], rq[MAXS / 2];
  __shared__ int perm[MAXS];
  __shared__ double red[32];
  __shared__ int s_sel[2];
  double* M = Msel + size_t(e) * s * s;

  if (active && !active[e]) {
    for (int i = threadIdx.x; i < s * s; i += blockDim.x) M[i] = 0.0;
    return;
  }
  const int Ne = s + (s & 1), half = Ne / 2;
  const double* Ge = G + size_t(e) * s * s;
  for (int idx = threadIdx.x; idx < Ne * Ne; idx += blockDim.x) {
    int i = idx % Ne, j = idx / Ne;
    A[i][j] = (i < s && j < s) ? 0.5 * (Ge[i + j * s] + Ge[j + i * s]) : 0.0;
    Q[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  // rotation floor: a rotation itself perturbs every rotated entry by ~eps*max_i a_ii, so
  // pairs below 1e-15*max_i a_ii (~4.5 eps) are decoupled as far as the rounding allows.
  // (A floor below the rounding level never terminates: 40 sweeps instead of 7-8 on the
  // rank-deficient, noisy C2 Grams.)  Relative accuracy of the tiny eigenpairs is neither
  // available from a Gram nor needed: pass 2 and the final SVD of C = U^T G make the basis exact.
  double dmax = 0.0;
  for (int i = threadIdx.x; i < s; i += blockDim.x) dmax = fmax(dmax, A[i][i]);
  const double afloor = fmax(1e-15 * block_max(dmax, red), 1e-300);
  __shared__ int s_rot;
  const int bk = threadIdx.x / half, bl = threadIdx.x % half;  // this thread's 2x2 block
  const bool has_blk = threadIdx.x < half * half;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < Ne - 1; ++r) {
      if (threadIdx.x < half) {
        int p, q;
        jacobi_pair(Ne, r, threadIdx.x, p, q);
        double c = 1.0, sn = 0.0;
        // rotate only pairs that are not yet decoupled to working precision
        if (fabs(A[p][q]) > 1e-16 * sqrt(fabs(A[p][p] * A[q][q])) && fabs(A[p][q]) > afloor) {
          sym_schur2(A[p][p], A[q][q], A[p][q], c, sn);
          s_rot = 1;
        }
        rp[threadIdx.x] = p; rq[threadIdx.x] = q; rc[threadIdx.x] = c; rs[threadIdx.x] = sn;
      }
      __syncthreads();
      if (has_blk) {
        const int pk = rp[bk], qk = rq[bk], pl = rp[bl], ql = rq[bl];
        const double ck = rc[bk], sk = rs[bk], cl = rc[bl], sl = rs[bl];
        const double a = A[pk][pl], b = A[pk][ql], c_ = A[qk][pl], d = A[qk][ql];
        // rows: r_p' = c r_p - s r_q, r_q' = s r_p + c r_q ; then the same on the columns
        const double a1 = ck * a - sk * c_, b1 = ck * b - sk * d, c1 = sk * a + ck * c_, d1 = sk * b + ck * d;
        double a2 = cl * a1 - sl * b1, b2 = sl * a1 + cl * b1, c2 = cl * c1 - sl * d1, d2 = sl * c1 + cl * d1;
        if (bk == bl && sk != 0.0) { b2 = 0.0; c2 = 0.0; }  // the annihilated pair (classical Jacobi)
        A[pk][pl] = a2; A[pk][ql] = b2; A[qk][pl] = c2; A[qk][ql] = d2;
      }
      for (int idx = threadIdx.x; idx < half * Ne; idx += blockDim.x) {  // Q <- Q J (column pairs)
        const int l = idx / Ne, j = idx % Ne, p = rp[l], q = rq[l];
        const double c = rc[l], sn = rs[l], qp = Q[j][p], qq = Q[j][q];
        Q[j][p] = c * qp - sn * qq;
        Q[j][q] = sn * qp + c * qq;
      }
      __syncthreads();
    }
    const int rotated = s_rot;
    __syncthreads();  // every thread has read s_rot before thread 0 resets it
    if (!rotated) break;
  }
  // descending order of the eigenvalues (stable rank sort, one thread per eigenvalue)
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    const double li = A[i][i];
    int rank = 0;
    for (int j = 0; j < s; ++j) {
      const double lj = A[j][j];
      rank += (lj > li) || (lj == li && j < i);
    }
    perm[rank] = i;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s; i += blockDim.x) lam_out[size_t(e) * s + i] = fmax(A[perm[i]][perm[i]], 0.0);
  for (int i = threadIdx.x; i < s * s; i += blockDim.x) M[i] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double smax = sqrt(fmax(A[perm[0]][perm[0]], 0.0));
    if (pass == 0) sigma1[e] = smax;
    const double thr = 0.5 * tau * sigma1[e];
    int o = off[e], kept = 0;
    for (int i = 0; i < s && o + kept < s; ++i) {
      double sg = sqrt(fmax(A[perm[i]][perm[i]], 0.0));
      if (!(sg > theta * smax) || !(sg > thr)) break;
      ++kept;
    }
    off[e] = o + kept;
    s_sel[0] = o;
    s_sel[1] = kept;
  }
  __syncthreads();
  const int o = s_sel[0], kept = s_sel[1];
  for (int idx = threadIdx.x; idx < kept * s; idx += blockDim.x) {
    int c = idx / s, i = idx % s;
    double sg = sqrt(fmax(A[perm[c]][perm[c]], 0.0));
    M[i + size_t(o + c) * s] = Q[i][perm[c]] / sg;
  }
}

// ---------------------------------------------------------------- deflating Cholesky-QR
// G: [E] N x N Gram (ld ldg, stride gs_e).  norm0 (nullable, diagonal read with ld ldn):
// squared norms of the columns before orthogonalisation against the previous basis; a column
// is deflated (dead) when G_kk <= defl^2 * norm0_k or G_kk == 0.
// PIVOTED Cholesky of the diagonally scaled Gram matrix: at each step the remaining column
// with the largest Schur-complement pivot is eliminated; elimination stops when the largest
// remaining scaled pivot is <= 1e-14 (those columns lie within 1e-7 of the span already
// built).  Tiny-but-accepted pivots are therefore processed last and cannot corrupt larger
// ones (the failure mode of unpivoted CholQR on nearly dependent Krylov blocks).
// With perm the pivot order, W[:, perm] = Q Rp (Rp upper triangular).  Outputs:
//   Rinv (N x N, ld N, stride N*N):  Q = W Rinv  (live new columns first, dead columns 0)
//   Rout (= R, or R * Rprev):  W = Q R with R[t][perm[a]] = Rp[t][a]  (column-permuted)
//   live flags: new column t is live iff t < number of accepted pivots.
__global__ void __launch_bounds__(PEXP_THREADS)
k_block_chol(int N, const double* G, long long gs_e, int ldg, const double* norm0, long long ns_e,
             int ldn, double defl, double* Rinv, const double* Rprev, long long rps_e, int ldrp, double* Rout,
             long long rs_e, int ldr, int* live, long long ls_e, const int* active, int pivoted, double piv_tol,
             double dtol, double* norm0_out, int* maskB, int* maskC) {
  const int e = blockIdx.x;
  if (active && !active[e]) {
    if (maskB && threadIdx.x == 0) { maskB[e] = 0; maskC[e] = 0; }
    return;
  }
  extern __shared__ double dsm[];
  double (*S)[MAXS + 1] = reinterpret_cast<double (*)[MAXS + 1]>(dsm);                       // scaled Gram / Schur
  double (*X)[MAXS + 1] = reinterpret_cast<double (*)[MAXS + 1]>(dsm + MAXS * (MAXS + 1));   // work
  __shared__ double d[MAXS];
  __shared__ double Lp[MAXS][MAXS + 1];  // Lp[a][t]: permuted lower factor (position a, pivot t)
  __shared__ int dead[MAXS], perm[MAXS], used[MAXS];
  __shared__ int s_np, s_j;
  __shared__ double s_piv, s_pmin;
  const double* Ge = G + e * gs_e;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    double g = Ge[k + size_t(k) * ldg];
    bool dk = !(g > 0.0);
    if (norm0 && !(g > defl * defl * norm0[e * ns_e + k + size_t(k) * ldn])) dk = true;
    dead[k] = dk;
    used[k] = 0;
    d[k] = g > 0.0 ? 1.0 / sqrt(g) : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    int i = idx % N, j = idx / N;
    S[i][j] = d[i] * d[j] * 0.5 * (Ge[i + size_t(j) * ldg] + Ge[j + size_t(i) * ldg]);
    Lp[i][j] = 0.0;
  }
  if (threadIdx.x == 0) { s_np = 0; s_pmin = INFINITY; }
  __syncthreads();
  for (int t = 0; t < N; ++t) {
    if (threadIdx.x == 0) {
      int jb = -1;
      double best = dtol > 0.0 ? dtol : piv_tol;
      if (pivoted) {
        for (int j = 0; j < N; ++j)
          if (!used[j] && !dead[j] && S[j][j] > best) { best = S[j][j]; jb = j; }
      } else {  // natural order (keeps the column order of an already well-conditioned block)
        for (int j = 0; j < N && jb < 0; ++j) {
          if (used[j] || dead[j]) continue;
          if (S[j][j] > best) { best = S[j][j]; jb = j; } else dead[j] = 1;
        }
      }
      s_j = jb;
      if (jb >= 0) {
        used[jb] = 1;
        perm[t] = jb;
        s_piv = sqrt(best);
        s_pmin = fmin(s_pmin, best);
        s_np = t + 1;
      }
    }
    __syncthreads();
    const int jb = s_j;
    if (jb < 0) break;
    const double pv = s_piv;
    // column of the factor for pivot t: l_i = S[i][jb] / pv for every not-yet-used column i
    for (int i = threadIdx.x; i < N; i += blockDim.x) X[i][0] = (i == jb) ? pv : (used[i] ? 0.0 : S[i][jb] / pv);
    __syncthreads();
    for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
      int i = idx % N, k = idx / N;
      if (!used[i] && !used[k]) S[i][k] -= X[i][0] * X[k][0];
    }
    // record l for every column (by original index) in slot t
    for (int i = threadIdx.x; i < N; i += blockDim.x) Lp[i][t] = X[i][0];
    __syncthreads();
  }
  const int np = s_np;
  // order: positions 0..np-1 = pivots, then the remaining columns in original order
  // (deferred mode: non-dead remaining columns are passed through raw at positions np..np+nd-1)
  __shared__ int s_nd;
  if (threadIdx.x == 0) {
    int q = np, nd = 0;
    if (dtol > 0.0)
      for (int j = 0; j < N; ++j)
        if (!used[j] && !dead[j]) { perm[q++] = j; ++nd; }
    for (int j = 0; j < N; ++j)
      if (!used[j] && (dtol <= 0.0 || dead[j])) perm[q++] = j;
    s_nd = nd;
  }
  __syncthreads();
  const int nd = s_nd;
  // masks of the follow-up stages of the in-block QR (pexp_api.cu inblock_qr): stage B (explicit
  // CGS2 of deferred columns) only when something was deferred; stage C (second CholQR) unless
  // every column was accepted with scaled pivots >= 1e-2 (same rule as the fused Arnoldi step)
  if (maskB && threadIdx.x == 0) {
    maskB[e] = nd > 0;
    maskC[e] = !(nd == 0 && np == N && s_pmin >= 1e-2);
  }
  // Rp[t][a] (upper, t <= a, t < np) = Lp[perm[a]][t];  X = Rp^{-1} on the leading np x np block
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    for (int k = 0; k < N; ++k) X[k][j] = 0.0;
    if (j < np) {
      for (int k = j; k >= 0; --k) {
        double sum = (k == j) ? 1.0 : 0.0;
        for (int q = k + 1; q <= j; ++q) sum -= Lp[perm[q]][k] * X[q][j];
        X[k][j] = sum / Lp[perm[k]][k];
      }
    }
  }
  __syncthreads();
  // Rinv[perm[a]][t] = d[perm[a]] * X[a][t]  (Q_t = sum_a W[:, perm[a]] Rinv[perm[a]][t])
  double* Ri = Rinv + size_t(e) * N * N;
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) Ri[idx] = 0.0;
  __syncthreads();
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    int a = idx % N, t = idx / N;
    Ri[perm[a] + size_t(t) * N] = d[perm[a]] * X[a][t];
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nd; q += blockDim.x) Ri[perm[np + q] + size_t(np + q) * N] = 1.0;  // raw copy
  if (live)
    for (int k = threadIdx.x; k < N; k += blockDim.x) live[e * ls_e + k] = k < np ? 1 : (k < np + nd ? 2 : 0);
  if (norm0_out && norm0)
    for (int k = threadIdx.x; k < N; k += blockDim.x)
      norm0_out[e * N + k] = norm0[e * ns_e + perm[k] + size_t(perm[k]) * ldn];
  __syncthreads();
  // R[t][c] = Lp[c][t] / d[c] for t < np (W[:, c] = sum_t Q_t R[t][c]); 0 if d[c] == 0
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    int t = idx % N, c = idx / N;
    X[t][c] = (t < np && d[c] > 0.0) ? Lp[c][t] / d[c] : 0.0;
  }
  __syncthreads();
  if (Rout) {
    double* Ro = Rout + e * rs_e;
    for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
      int k = idx % N, j = idx / N;
      double v;
      if (Rprev) {
        const double* Rp = Rprev + e * rps_e;
        v = 0.0;
        for (int p = 0; p < N; ++p) v += X[k][p] * Rp[p + size_t(j) * ldrp];
      } else {
        v = X[k][j];
      }
      Ro[k + size_t(j) * ldr] = v;
    }
  }
}

// Correction for deferred columns (class 2) against accepted orthonormal columns (class 1):
// Mc[a][k] = -Gb[a][k] for a in A, k in D (so that Block += Block * Mc is one CGS step).
__global__ void k_defer_corr(int N, const double* Gb, long long gs_e, const int* cls, long long cs_e, double* Mc,
                             const int* active, int plus_identity) {
  const int e = blockIdx.x;
  if (active && !active[e]) return;
  const int* c = cls + e * cs_e;
  const double* G = Gb + e * gs_e;
  double* M = Mc + size_t(e) * N * N;
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    int a = idx % N, k = idx / N;
    M[idx] = ((c[a] == 1 && c[k] == 2) ? -G[a + size_t(k) * N] : 0.0) + (plus_identity && a == k ? 1.0 : 0.0);
  }
}

void launch_defer_corr(cudaStream_t st, int E, int N, const double* Gb, long long gs_e, const int* cls, long long cs_e,
                       double* Mc, const int* active, bool plus_identity) {
  ProfScope ps(PC_SVDSMALL, st, 0.0, 0.0);
  k_defer_corr<<<E, 128, 0, st>>>(N, Gb, gs_e, cls, cs_e, Mc, active, plus_identity ? 1 : 0);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- one-sided Jacobi SVD
// C: [E] s x s col-major; rows 0..kk-1 are the coefficients U^T G of the current basis.
// Produces Qs (s x s, columns = left singular vectors of C, sorted by sigma desc),
// sig [E][s], Cs (s x s: row c = sigma_c * v_c^T) and m[e] = #{sigma > tau*sigma_1}.
__global__ void __launch_bounds__(PEXP_THREADS)
k_onesided_svd(int s, const double* C, const int* kk_arr, double tau, double* Qs, double* sig,
               double* Cs, int* m_out, const int* active) {
  const int e = blockIdx.x;
  extern __shared__ double dsm[];
  double (*W)[MAXS + 1] = reinterpret_cast<double (*)[MAXS + 1]>(dsm);  // W[j][i] = row j of C
  double (*Q)[MAXS + 1] = reinterpret_cast<double (*)[MAXS + 1]>(dsm + MAXS * (MAXS + 1));
  __shared__ double nrm[MAXS];
  __shared__ int perm[MAXS];
  __shared__ int s_conv;
  if (active && !active[e]) {
    if (threadIdx.x == 0) m_out[e] = 0;
    return;
  }
  const int kk = kk_arr[e];
  const int Ne = kk + (kk & 1);
  const double* Ce = C + size_t(e) * s * s;
  for (int idx = threadIdx.x; idx < MAXS * MAXS; idx += blockDim.x) {
    int j = idx / MAXS, i = idx % MAXS;
    W[j][i] = (j < kk && i < s) ? Ce[j + size_t(i) * s] : 0.0;
    Q[j][i] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int g = threadIdx.x / 8, lg = threadIdx.x % 8;  // 32 groups of 8 lanes
  for (int sweep = 0; sweep < 60 && Ne >= 2; ++sweep) {
    if (threadIdx.x == 0) s_conv = 1;
    __syncthreads();
    for (int r = 0; r < Ne - 1; ++r) {
      const bool act = g < Ne / 2;
      int p = 0, q = 0;
      if (act) jacobi_pair(Ne, r, g, p, q);
      double al = 0.0, be = 0.0, ga = 0.0;
      if (act)
        for (int i = lg; i < s; i += 8) {
          double wp = W[p][i], wq = W[q][i];
          al += wp * wp; be += wq * wq; ga += wp * wq;
        }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {  // reduce within the 8-lane group (all lanes execute)
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      if (act && fabs(ga) > 1e-15 * sqrt(al * be) && fabs(ga) > 1e-300) {
        if (lg == 0) s_conv = 0;
        double zeta = (be - al) / (2.0 * ga);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
        double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int i = lg; i < s; i += 8) {
          double wp = W[p][i], wq = W[q][i];
          W[p][i] = c * wp - sn * wq;
          W[q][i] = sn * wp + c * wq;
        }
        for (int i = lg; i < kk; i += 8) {
          double qp = Q[i][p], qq = Q[i][q];
          Q[i][p] = c * qp - sn * qq;
          Q[i][q] = sn * qp + c * qq;
        }
      }
      __syncthreads();
    }
    if (s_conv) break;
    __syncthreads();
  }
  for (int j = threadIdx.x; j < MAXS; j += blockDim.x) {
    double a = 0.0;
    if (j < kk)
      for (int i = 0; i < s; ++i) a += W[j][i] * W[j][i];
    nrm[j] = sqrt(a);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < s; ++i) perm[i] = i;
    for (int i = 0; i < kk; ++i) {
      int b = i;
      for (int j = i + 1; j < kk; ++j)
        if (nrm[perm[j]] > nrm[perm[b]]) b = j;
      int t = perm[i]; perm[i] = perm[b]; perm[b] = t;
    }
    int m = 0;
    double s1 = kk > 0 ? nrm[perm[0]] : 0.0;
    if (s1 > 0.0)
      for (int i = 0; i < kk; ++i)
        if (nrm[perm[i]] > tau * s1) ++m;
    m_out[e] = m;
  }
  __syncthreads();
  double* Qe = Qs + size_t(e) * s * s;
  double* Ce2 = Cs + size_t(e) * s * s;
  for (int idx = threadIdx.x; idx < s * s; idx += blockDim.x) {
    int i = idx % s, c = idx / s;  // Qe[i + c*s] = Q[i][perm[c]]
    Qe[idx] = (c < kk && i < kk) ? Q[i][perm[c]] : 0.0;
    // Ce2 row c, column i  (col-major s x s: Ce2[c + i*s])
    int cc = idx % s, ii = idx / s;
    Ce2[cc + size_t(ii) * s] = (cc < kk) ? W[perm[cc]][ii] : 0.0;
  }
  for (int c = threadIdx.x; c < s; c += blockDim.x) sig[size_t(e) * s + c] = c < kk ? nrm[perm[c]] : 0.0;
}

// Msel_e (s x mmax) = Qs[:, :mmax] restricted to kk columns with nonzero sigma; Cfin_e (mmax x s)
// = rows c < m_e of Cs, zero otherwise; fill[e*mmax + c] = 1 where U_final column c must be
// replaced by a (pseudo-random, then orthonormalised) padding vector.
__global__ void k_build_final(int s, int mmax, const int* kk_arr, const double* Qs, const double* sig,
                              const double* Cs, const int* m_arr, double* Msel, double* Cfin, int* fill) {
  const int e = blockIdx.x;
  const int kk = kk_arr[e], m = m_arr[e];
  const double* Qe = Qs + size_t(e) * s * s;
  const double* Ce = Cs + size_t(e) * s * s;
  double* Me = Msel + size_t(e) * s * mmax;
  double* Fe = Cfin + size_t(e) * mmax * s;
  for (int idx = threadIdx.x; idx < s * mmax; idx += blockDim.x) {
    int i = idx % s, c = idx / s;
    bool ok = c < kk && sig[size_t(e) * s + c] > 0.0;
    Me[idx] = ok ? Qe[i + size_t(c) * s] : 0.0;
    int cr = idx % mmax, ic = idx / mmax;  // Cfin col-major mmax x s
    Fe[cr + size_t(ic) * mmax] = (cr < m) ? Ce[cr + size_t(ic) * s] : 0.0;
  }
  for (int c = threadIdx.x; c < mmax; c += blockDim.x)
    fill[e * mmax + c] = !(c < kk && sig[size_t(e) * s + c] > 0.0);
}

// ---------------------------------------------------------------- Chebyshev interpolant pieces
// node_rule 1: coef_e[i][q][c] = sum_k Dmat[(i*nq + q)*s + k] * Cfin_e[c][k]  (Cfin col-major mmax x s:
// the coefficient rows at the Chebyshev-Lobatto nodes);  crit[e] = eta * max_k ||Cfin[:, k]||.
__global__ void k_poly_coef(int s, int mmax, int nq, const double* Dmat, const double* Cfin, double eta,
                            double* coef, double* crit) {
  const int e = blockIdx.x;
  extern __shared__ double sm[];
  double* Y = sm;  // [s][mmax] (as stored)
  __shared__ double red[32];
  const double* Ce = Cfin + size_t(e) * mmax * s;
  for (int idx = threadIdx.x; idx < mmax * s; idx += blockDim.x) Y[idx] = Ce[idx];
  __syncthreads();
  double* ce = coef + size_t(e) * (s - 1) * nq * mmax;
  for (int idx = threadIdx.x; idx < (s - 1) * nq * mmax; idx += blockDim.x) {
    const int c = idx % mmax, iq = idx / mmax;
    const double* Dr = Dmat + size_t(iq) * s;
    double a = 0.0;
    for (int k = 0; k < s; ++k) a = fma(Dr[k], Y[c + k * mmax], a);
    ce[idx] = a;
  }
  double mx = 0.0;
  for (int k = threadIdx.x; k < s; k += blockDim.x) {
    double a = 0.0;
    for (int c = 0; c < mmax; ++c) a += Y[c + k * mmax] * Y[c + k * mmax];
    mx = fmax(mx, sqrt(a));
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) crit[e] = eta * mx;
}

// ---------------------------------------------------------------- not-a-knot spline
// Kinv: inverse of the s x s not-a-knot second-derivative system (host-computed, depends
// only on s).  Cfin_e: mmax x s samples.  coef_e: [s-1][4][mmax] Taylor coefficients
// (p, p', p'', p''') at the left node of each piece; crit[e] = eta * max_i ||Cfin[:, i]||.
__global__ void k_spline(int s, int mmax, const double* Kinv, const double* Cfin, double h, double eta,
                         double* coef, double* crit, const int* active) {
  const int e = blockIdx.x;
  extern __shared__ double sm[];
  double* Y = sm;              // [mmax][s]
  double* R = sm + mmax * s;   // [mmax][s]
  double* Mv = R + mmax * s;   // [mmax][s]
  __shared__ double red[32];
  const double* Ce = Cfin + size_t(e) * mmax * s;
  for (int idx = threadIdx.x; idx < mmax * s; idx += blockDim.x) {
    int c = idx / s, i = idx % s;
    Y[idx] = Ce[c + size_t(i) * mmax];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < mmax * s; idx += blockDim.x) {
    int c = idx / s, i = idx % s;
    R[idx] = (i == 0 || i == s - 1) ? 0.0 : 6.0 * (Y[c * s + i + 1] - 2.0 * Y[c * s + i] + Y[c * s + i - 1]) / (h * h);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < mmax * s; idx += blockDim.x) {
    int c = idx / s, i = idx % s;
    double a = 0.0;
    for (int k = 0; k < s; ++k) a += Kinv[i + k * s] * R[c * s + k];
    Mv[idx] = a;
  }
  __syncthreads();
  double* ce = coef + size_t(e) * (s - 1) * 4 * mmax;
  for (int idx = threadIdx.x; idx < mmax * (s - 1); idx += blockDim.x) {
    int c = idx % mmax, i = idx / mmax;
    double y0 = Y[c * s + i], y1 = Y[c * s + i + 1], m0 = Mv[c * s + i], m1 = Mv[c * s + i + 1];
    double* o = ce + size_t(i) * 4 * mmax;
    o[0 * mmax + c] = y0;
    o[1 * mmax + c] = (y1 - y0) / h - h * (2.0 * m0 + m1) / 6.0;
    o[2 * mmax + c] = m0;
    o[3 * mmax + c] = (m1 - m0) / h;
  }
  double mx = 0.0;
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    double a = 0.0;
    for (int c = 0; c < mmax; ++c) a += Y[c * s + i] * Y[c * s + i];
    mx = fmax(mx, sqrt(a));
  }
  mx = block_max(mx, red);
  if (threadIdx.x == 0) crit[e] = eta * mx;
  (void)active;
}

// ---------------------------------------------------------------- projected SaI problem
// One cluster per evaluation.  Current cycle: A_hat = (I - H^{-1})/gamma on the live columns.
// With restarts the completed cycles precede it (NA, D x D) and feed it through the coupling
// rows CPL into its block-0 coordinates; the full system
//     [z_old; z]' = [[NA, 0], [CPL, A_hat]] [z_old; z] + E_1 p(t)      (forced: rows [0, m))
// is integrated exactly over the s-1 cubic pieces with ONE Pade-13 expm of the augmented
// matrix (size D + Kp + 4m).  The residual is the current cycle's (it is the residual of the
// whole accumulated approximation).
__global__ void __launch_bounds__(PEXP_THREADS, SMALL_MINB) k_small_problem(SPArgs a) {
  __shared__ int idx[KSMALL_MAX];
  __shared__ int tidx[MAXS], lpos[MAXS];
  __shared__ int s_K, s_mt, s_ml;
  __shared__ double red[32];
  extern __shared__ double zsm[];  // SP_DYN bytes: chaining state, partials, F slice
  const Grp g = this_grp();
  const int slot = blockIdx.x / g.size, nslot = gridDim.x / g.size;
  double* S0 = a.work + slot * a.work_slot;
  const int ld = a.Nmax;
  const size_t MM = size_t(ld) * ld;
  double* S1 = S0 + MM;
  double* S2 = S1 + MM;
  double* WK = S2 + MM;
  int* piv = a.iwork + slot * a.iwork_slot;
  const int K = a.K, m = a.m;
  for (int e = slot; e < a.E; e += nslot) {
    if (a.active && !a.active[e]) continue;
    const double* He = a.H + e * a.hs_e;
    const int* lv = a.live + e * a.ls_e;
    if (threadIdx.x == 0) {
      int k = 0;
      for (int c = 0; c < K; ++c)
        if (lv[c]) idx[k++] = c;
      s_K = k;
      int mt = 0;
      for (int c = K; c < K + m; ++c)
        if (lv[c]) tidx[mt++] = c;
      s_mt = mt;
      int ml = 0;
      for (int r = 0; r < k; ++r)
        if (idx[r] >= K - m) lpos[ml++] = r;
      s_ml = ml;
    }
    __syncthreads();
    const int Kp = s_K, mt = s_mt, ml = s_ml;
    const double gam = a.gam[e];
    const int forced = a.kind == 0;
    const int D = a.Dn ? a.Dn[e] : 0;
    const int Kl = a.Kl ? a.Kl[e] : 0;
    const int Dz = D + Kp;
    const int nq = a.nq;
    const int Nn = Dz + (forced ? nq * m : 0);
    double* NAe = a.NA ? a.NA + e * a.nas_e : nullptr;
    const double* CPe = a.CPL ? a.CPL + e * a.cpls_e : nullptr;
    // Hs -> S0, Hinv -> S1
    for (int t = threadIdx.x + g.rank * blockDim.x; t < Kp * Kp; t += blockDim.x * g.size) {
      int i = t % Kp, j = t / Kp;
      S0[i + size_t(j) * ld] = He[idx[i] + size_t(idx[j]) * a.ldh];
    }
    grp_sync(g);
    cta_identity(Kp, S1, ld, 1.0, g);
    cta_lu(Kp, S0, ld, piv, red, g, zsm, int(SP_DYN / 8));
    cta_lu_solve(Kp, S0, ld, piv, S1, ld, Kp, g, zsm, int(SP_DYN / 8), true);
    // augmented matrix (times h) in S2; on a restart check the new cycle is appended to NA
    const bool wr = a.restart_write && NAe;
    for (int t = threadIdx.x + g.rank * blockDim.x; t < Nn * Nn; t += blockDim.x * g.size) {
      int i = t % Nn, j = t / Nn;
      double v = 0.0;
      if (j >= Dz) {
        if (forced && i < m && j - Dz == i) v = 1.0;  // h E_1: forcing into cycle 0, block 0
      } else if (i < D && j < D) {
        v = NAe[i + size_t(j) * a.na_ld];
      } else if (i >= D && i < Dz) {
        const int r = i - D;
        if (j >= D && j < Dz) {
          v = ((r == j - D ? 1.0 : 0.0) - S1[r + size_t(j - D) * ld]) / gam;
          if (wr) NAe[i + size_t(j) * a.na_ld] = v;
        } else if (j >= D - Kl && j < D && idx[r] < m) {
          v = CPe[idx[r] + size_t(j - (D - Kl)) * m];
          if (wr) NAe[i + size_t(j) * a.na_ld] = v;
        }
      }
      // polynomial chain: unscaled identity blocks (the h^q factors are applied in the chain)
      if (forced && i >= Dz && j - i == m && i < Dz + (nq - 1) * m) S2[i + size_t(j) * ld] = 1.0;
      else S2[i + size_t(j) * ld] = a.h * v;
    }
    if (wr && g.rank == 0) {  // TX = (1/gamma) H_tail X, X = last-block rows of H^{-1}
      double* TXe = a.TX + e * (long long)m * a.kcap;
      for (int t = threadIdx.x; t < m * Kp; t += blockDim.x) {
        const int j = t % m, r = t / m;
        double v = 0.0;
        if (lv[K + j])
          for (int c = 0; c < ml; ++c) v = fma(He[K + j + size_t(idx[lpos[c]]) * a.ldh], S1[lpos[c] + size_t(r) * ld], v);
        TXe[j + size_t(r) * m] = v / gam;
      }
    }
    if (a.kplast && g.rank == 0 && threadIdx.x == 0) a.kplast[e] = Kp;
    grp_sync(g);
    cta_expm_pade13(Nn, S2, ld, WK, ld, piv, red, g, zsm, int(SP_DYN / 8));
    // ---- exact chaining over the np pieces (rows split over the group, one group barrier per
    // piece): z_{i+1} = F z_i + f_i with F = e^{h N}[0:Dz, 0:Dz] and the piece forcing
    // f_i = sum_q h^q B_q c_{i,q}; the state is replicated in every CTA's shared memory (each CTA
    // publishes its rows through DSMEM).  Residual at every node (DESIGN.md §3 #6): ts = R z[D:],
    // R = H_tail H^{-1}[last block rows, :] (mt x Kp), reduced per piece from per-CTA partials.
    {
      cg::cluster_group cl = cg::this_cluster();
      const int np = a.npieces ? a.npieces[e] : a.npieces_const;
      const int rs = (Dz + g.size - 1) / g.size;
      const int r0 = min(Dz, g.rank * rs), nr = min(Dz, r0 + rs) - r0;
      const int nrt = (nr + 31) / 32, jp = max(1, (PEXP_THREADS / 32) / max(nrt, 1)), jper = (Dz + jp - 1) / jp;
      double* zb0 = zsm;
      double* zb1 = zsm + KSMALL_MAX;
      double* psum = zsm + 2 * KSMALL_MAX;  // [jp][nrt*32]
      double* zown = psum + CH_PSUM;        // [nr]
      double* ring = zown + KSMALL_MAX;     // [RING_N][MAXS] per-piece residual partials (read by rank 0)
      double* Fs = ring + RING_N * MAXS;    // own rows of F, column-major (ld nr), if they fit
      const bool ring_all = np <= RING_N;   // keep every piece's partial: reduce after the chain
      const bool fsm = size_t(nr) * Dz <= FS_CAP;
      double* Fo = WK;                      // [np][Dz] forcing of every piece
      double* Rg = WK + size_t(np) * Dz;    // [mt][Kp]
      double* Ze = a.Z + e * a.zs_e;
      const double* cf = forced ? a.coef + size_t(e) * (a.s - 1) * nq * m : nullptr;
      for (int t = threadIdx.x + g.rank * blockDim.x; t < a.nout * a.kcap; t += blockDim.x * g.size) Ze[t] = 0.0;
      if (forced)
        for (int t = threadIdx.x; t < nr * np; t += blockDim.x) {
          const int r = r0 + t % nr, i = t / nr;
          const double* ci = cf + size_t(i) * nq * m;
          double v = 0.0, hq = 1.0;
          for (int q = 0; q < nq; ++q) {
            const double* B = S2 + size_t(Dz + q * m) * ld;
            double acc = 0.0;
            for (int c = 0; c < m; ++c) acc = fma(B[r + size_t(c) * ld], ci[q * m + c], acc);
            v = fma(hq, acc, v);
            hq *= a.h;
          }
          Fo[size_t(i) * Dz + r] = v;
        }
      for (int t = threadIdx.x; t < mt * nr; t += blockDim.x) {
        const int r = r0 + t % nr, tc = t / nr;
        if (r < D) continue;
        const int j = r - D;
        double v = 0.0;
        for (int c = 0; c < ml; ++c)
          v = fma(He[tidx[tc] + size_t(idx[lpos[c]]) * a.ldh], S1[lpos[c] + size_t(j) * ld], v);
        Rg[size_t(tc) * Kp + j] = v;
      }
      if (fsm)
        for (int t = threadIdx.x; t < nr * Dz; t += blockDim.x) {
          const int rl = t % nr, j = t / nr;
          Fs[t] = S2[r0 + rl + size_t(j) * ld];
        }
      for (int r = threadIdx.x; r < Dz; r += blockDim.x) zb0[r] = (!forced && r == 0) ? a.beta[e] : 0.0;
      grp_sync(g);
      for (int rl = threadIdx.x; rl < nr; rl += blockDim.x)
        if (r0 + rl >= D) Ze[idx[r0 + rl - D]] = zb0[r0 + rl];
      const double* Fp = fsm ? Fs : S2 + r0;
      const int ldf = fsm ? nr : ld;
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      double maxres = 0.0;
      __shared__ double tsum[MAXS];
      for (int i = 0; i < np; ++i) {
        const double* cur = (i & 1) ? zb1 : zb0;
        double* nxt = (i & 1) ? zb0 : zb1;
        for (int task = warp; task < nrt * jp; task += PEXP_THREADS / 32) {
          const int rt = task % nrt, p = task / nrt, rl = rt * 32 + lane;
          const int j0 = p * jper, j1 = min(Dz, j0 + jper);
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          if (rl < nr) {
            const double* fr = Fp + rl;
            int j = j0;
            for (; j + 3 < j1; j += 4) {
              s0 = fma(fr[size_t(j) * ldf], cur[j], s0);
              s1 = fma(fr[size_t(j + 1) * ldf], cur[j + 1], s1);
              s2 = fma(fr[size_t(j + 2) * ldf], cur[j + 2], s2);
              s3 = fma(fr[size_t(j + 3) * ldf], cur[j + 3], s3);
            }
            for (; j < j1; ++j) s0 = fma(fr[size_t(j) * ldf], cur[j], s0);
          }
          psum[p * nrt * 32 + rl] = (s0 + s1) + (s2 + s3);
        }
        __syncthreads();
        const int node = i + 1;
        const bool out = node % a.out_stride == 0 && node / a.out_stride < a.nout;
        for (int rl = threadIdx.x; rl < nr; rl += blockDim.x) {
          double v = forced ? Fo[size_t(i) * Dz + r0 + rl] : 0.0;
          for (int p = 0; p < jp; ++p) v += psum[p * nrt * 32 + rl];
          zown[rl] = v;
          for (int q = 0; q < g.size; ++q) (g.size > 1 ? cl.map_shared_rank(nxt, q) : nxt)[r0 + rl] = v;
          if (out && r0 + rl >= D) Ze[size_t(node / a.out_stride) * a.kcap + idx[r0 + rl - D]] = v;
        }
        __syncthreads();
        if (mt > 0)
          for (int tc = warp; tc < mt; tc += PEXP_THREADS / 32) {
            double sacc = 0.0;
            for (int rl = lane; rl < nr; rl += 32)
              if (r0 + rl >= D) sacc = fma(Rg[size_t(tc) * Kp + r0 + rl - D], zown[rl], sacc);
            sacc = warp_sum(sacc);
            if (lane == 0) ring[(ring_all ? i : (i & 1)) * MAXS + tc] = sacc;
          }
        grp_sync(g);
        if (!ring_all && g.rank == 0 && mt > 0) {  // residual of node i+1 (partials stable until the next barrier)
          for (int tc = threadIdx.x; tc < mt; tc += blockDim.x) {
            double v = 0.0;
            for (int q = 0; q < g.size; ++q) v += (g.size > 1 ? cl.map_shared_rank(ring, q) : ring)[(i & 1) * MAXS + tc];
            tsum[tc] = v;
          }
          __syncthreads();
          if (threadIdx.x == 0) {
            double r2 = 0.0;
            if (a.stop_rule == 1) {  // ||(I - gamma A) Vtail t||^2 = t^T Gt t
              const double* Gt = a.Gt + e * a.gts_e;
              for (int i1 = 0; i1 < mt; ++i1)
                for (int i2 = 0; i2 < mt; ++i2)
                  r2 += tsum[i1] * Gt[(tidx[i1] - K) + size_t(tidx[i2] - K) * m] * tsum[i2];
            } else {                 // ||Vtail t||^2 = ||t||^2 (orthonormal tail)
              for (int i1 = 0; i1 < mt; ++i1) r2 += tsum[i1] * tsum[i1];
            }
            maxres = fmax(maxres, sqrt(fmax(r2, 0.0)) / gam);
          }
        }
      }
      if (ring_all && g.rank == 0 && mt > 0) {  // residuals of all nodes after the chain (one thread per node)
        double mr = 0.0;
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
          double ts[MAXS];
          for (int tc = 0; tc < mt; ++tc) {
            double v = 0.0;
            for (int q = 0; q < g.size; ++q) v += (g.size > 1 ? cl.map_shared_rank(ring, q) : ring)[i * MAXS + tc];
            ts[tc] = v;
          }
          double r2 = 0.0;
          if (a.stop_rule == 1) {
            const double* Gt = a.Gt + e * a.gts_e;
            for (int i1 = 0; i1 < mt; ++i1)
              for (int i2 = 0; i2 < mt; ++i2) r2 += ts[i1] * Gt[(tidx[i1] - K) + size_t(tidx[i2] - K) * m] * ts[i2];
          } else {
            for (int i1 = 0; i1 < mt; ++i1) r2 += ts[i1] * ts[i1];
          }
          mr = fmax(mr, sqrt(fmax(r2, 0.0)) / gam);
        }
        mr = block_max(mr, red);
        if (threadIdx.x == 0) maxres = mr;
      }
      if (g.rank == 0 && threadIdx.x == 0) {
        a.res[e] = maxres;
        int cv = (mt == 0) || (maxres <= a.crit[e]);
        a.conv[e] = cv;
        if (cv && a.kfin) a.kfin[e] = K;
      }
    }  // rank 0
    grp_sync(g);
  }
}

// Finish a restart for the still-active evaluations: CPL = R TX (R = Q^T W0 of the new
// block 0), D += width of the closed cycle, fresh H and live flags for the new cycle.
__global__ void k_restart_finish(int E, int m, int kcap, const double* R, const double* TX, double* CPL,
                                 int* Dn, int* Kl, const int* kplast, double* H, long long hs_e, int* live,
                                 const int* active) {
  const int e = blockIdx.x;
  if (active && !active[e]) return;
  const int kp = kplast[e];
  const double* Re = R + size_t(e) * m * m;
  const double* Te = TX + size_t(e) * m * kcap;
  double* Ce = CPL + size_t(e) * m * kcap;
  for (int t = threadIdx.x; t < m * kp; t += blockDim.x) {
    const int i = t % m, r = t / m;
    double v = 0.0;
    for (int j = 0; j < m; ++j) v = fma(Re[i + size_t(j) * m], Te[j + size_t(r) * m], v);
    Ce[i + size_t(r) * m] = v;
  }
  double* He = H + e * hs_e;
  for (long long t = threadIdx.x; t < hs_e; t += blockDim.x) He[t] = 0.0;
  for (int c = threadIdx.x + m; c < kcap; c += blockDim.x) live[size_t(e) * kcap + c] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    Dn[e] += kp;
    Kl[e] = kp;
  }
}

void launch_restart_finish(cudaStream_t st, int E, int m, int kcap, const double* R, const double* TX, double* CPL,
                           int* Dn, int* Kl, const int* kplast, double* H, long long hs_e, int* live,
                           const int* active) {
  ProfScope ps(PC_SMALL, st, 0.0, 0.0);
  k_restart_finish<<<E, PEXP_THREADS, 0, st>>>(E, m, kcap, R, TX, CPL, Dn, Kl, kplast, H, hs_e, live, active);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- grouped homogeneous legs
// One CTA per group of m legs (kind 2).  Block 0 of the Krylov basis is the QR of the legs'
// start vectors v_j(T_{j+1}) = Q R0, so z_c(0) = R0[:, c].  With F = exp(dT * A_hat) the
// projected states z_c(q dT) = F^q z_c(0) are advanced together (one K x K x m GEMM per step);
// the contribution of leg j = j0 + c to output i = j + q (q >= 1) is accumulated in
// Zsum[e][i] (K-vectors), so that Yh_e[i] = V_e Zsum[e][i] is the group's share of
// sum_{j<i} exp((T_{i+1} - T_{j+1}) A) v_j(T_{j+1}) (Eq.(superposition)).
// Residual per leg and step (SaI form) against crit_c; convergence when every leg passes.
__global__ void __launch_bounds__(PEXP_THREADS, SMALL_MINB) k_small_hom(SPArgs a) {
  extern __shared__ double hsm[];  // HOM_DYN bytes: LU scratch; later residual ring + F slice
  __shared__ int idx[KSMALL_MAX];
  __shared__ int tidx[MAXS], lpos[MAXS];
  __shared__ int s_K, s_mt, s_ml;
  __shared__ double red[32];
  const Grp g = this_grp();
  const int slot = blockIdx.x / g.size, nslot = gridDim.x / g.size;
  double* S0 = a.work + slot * a.work_slot;
  const int ld = a.Nmax;
  const size_t MM = size_t(ld) * ld;
  double* S1 = S0 + MM;
  double* S2 = S1 + MM;
  double* WK = S2 + MM;
  int* piv = a.iwork + slot * a.iwork_slot;
  const int K = a.K, m = a.m;
  for (int e = slot; e < a.E; e += nslot) {
    if (a.active && !a.active[e]) continue;
    const double* He = a.H + e * a.hs_e;
    const int* lv = a.live + e * a.ls_e;
    if (threadIdx.x == 0) {
      int k = 0;
      for (int c = 0; c < K; ++c)
        if (lv[c]) idx[k++] = c;
      s_K = k;
      int mt = 0;
      for (int c = K; c < K + m; ++c)
        if (lv[c]) tidx[mt++] = c;
      s_mt = mt;
      int ml = 0;
      for (int r = 0; r < k; ++r)
        if (idx[r] >= K - m) lpos[ml++] = r;
      s_ml = ml;
    }
    __syncthreads();
    const int Kp = s_K, mt = s_mt, ml = s_ml;
    const double gam = a.gam[e];
    for (int t = threadIdx.x + g.rank * blockDim.x; t < Kp * Kp; t += blockDim.x * g.size) {
      int i = t % Kp, j = t / Kp;
      S0[i + size_t(j) * ld] = He[idx[i] + size_t(idx[j]) * a.ldh];
    }
    grp_sync(g);
    cta_identity(Kp, S1, ld, 1.0, g);
    cta_lu(Kp, S0, ld, piv, red, g, hsm, int(HOM_DYN / 8));
    cta_lu_solve(Kp, S0, ld, piv, S1, ld, Kp, g, hsm, int(HOM_DYN / 8), true);
    for (int t = threadIdx.x + g.rank * blockDim.x; t < Kp * Kp; t += blockDim.x * g.size) {
      int i = t % Kp, j = t / Kp;
      S2[i + size_t(j) * ld] = a.h * ((i == j ? 1.0 : 0.0) - S1[i + size_t(j) * ld]) / gam;
    }
    grp_sync(g);
    cta_expm_pade13(Kp, S2, ld, WK, ld, piv, red, g, hsm, int(HOM_DYN / 8));
    // ---- propagation Z_q = F Z_{q-1} (Kp x m), rows split over the group, one group barrier
    // per step.  The replicated state lives in the slot's global workspace (L2; read with
    // __ldcg across CTAs), each CTA accumulates its own rows of every leg's outputs and a partial
    // of the residual ts = R Z_q (R = H_tail H^{-1}[last block rows, :], mt x Kp) per leg.
    cg::cluster_group cl = cg::this_cluster();
    const int rs = (Kp + g.size - 1) / g.size;
    const int r0 = min(Kp, g.rank * rs), nr = min(Kp, r0 + rs) - r0;
    double* Zb0 = WK;                          // [m][Kp]
    double* Zb1 = WK + size_t(Kp) * m;         // [m][Kp]
    double* Rg = Zb1 + size_t(Kp) * m;         // [mt][Kp]
    double* zown = Rg + size_t(mt) * Kp;       // [m][nr] per CTA (disjoint rows)
    double* ring = hsm;                        // [2][16*16]
    double* Fs = hsm + 2 * 256;                // own rows of F, column-major (ld nr), if they fit
    const bool fsm = size_t(nr) * Kp <= HOM_FS_CAP;
    const double* R0 = a.R0 + size_t(e) * m * m;
    double* Ze = a.Z + e * a.zs_e;
    for (int t = threadIdx.x; t < nr * m; t += blockDim.x) {
      const int r = r0 + t % nr, c = t / nr;
      Zb0[r + size_t(c) * Kp] = idx[r] < m ? R0[idx[r] + c * m] : 0.0;
    }
    for (int t = threadIdx.x + g.rank * blockDim.x; t < a.nout * a.kcap; t += blockDim.x * g.size) Ze[t] = 0.0;
    for (int t = threadIdx.x; t < mt * nr; t += blockDim.x) {
      const int j = r0 + t % nr, tc = t / nr;
      double v = 0.0;
      for (int c = 0; c < ml; ++c)
        v = fma(He[tidx[tc] + size_t(idx[lpos[c]]) * a.ldh], S1[lpos[c] + size_t(j) * ld], v);
      Rg[size_t(tc) * Kp + j] = v;
    }
    if (fsm)
      for (int t = threadIdx.x; t < nr * Kp; t += blockDim.x) Fs[t] = S2[r0 + t % nr + size_t(t / nr) * ld];
    grp_sync(g);
    const double* Fp = fsm ? Fs : S2 + r0;
    const int ldf = fsm ? nr : ld;
    const int j0 = (e % a.groups) * m;
    const double* cc = a.critc + size_t(e) * m;
    const int* hc = a.horc + size_t(e) * m;
    int qmax = 0;
    for (int c = 0; c < m; ++c) qmax = max(qmax, hc[c]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double worst = 0.0;
    for (int q = 1; q <= qmax; ++q) {
      const double* cur = (q & 1) ? Zb0 : Zb1;
      double* nxt = (q & 1) ? Zb1 : Zb0;
      for (int t = threadIdx.x; t < nr * m; t += blockDim.x) {
        const int rl = t % nr, c = t / nr;
        const double* fr = Fp + rl;
        const double* zc = cur + size_t(c) * Kp;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int j = 0;
        for (; j + 3 < Kp; j += 4) {
          s0 = fma(fr[size_t(j) * ldf], __ldcg(zc + j), s0);
          s1 = fma(fr[size_t(j + 1) * ldf], __ldcg(zc + j + 1), s1);
          s2 = fma(fr[size_t(j + 2) * ldf], __ldcg(zc + j + 2), s2);
          s3 = fma(fr[size_t(j + 3) * ldf], __ldcg(zc + j + 3), s3);
        }
        for (; j < Kp; ++j) s0 = fma(fr[size_t(j) * ldf], __ldcg(zc + j), s0);
        const double v = (s0 + s1) + (s2 + s3);
        __stcg(nxt + r0 + rl + size_t(c) * Kp, v);
        zown[r0 + rl + size_t(c) * Kp] = v;
        if (q <= hc[c]) Ze[size_t(j0 + c + q) * a.kcap + idx[r0 + rl]] += v;
      }
      __syncthreads();
      if (mt > 0)
        for (int pr = warp; pr < mt * m; pr += PEXP_THREADS / 32) {
          const int tc = pr % mt, c = pr / mt;
          double sacc = 0.0;
          if (q <= hc[c])
            for (int rl = lane; rl < nr; rl += 32)
              sacc = fma(Rg[size_t(tc) * Kp + r0 + rl], zown[r0 + rl + size_t(c) * Kp], sacc);
          sacc = warp_sum(sacc);
          if (lane == 0) ring[(q & 1) * 256 + pr] = sacc;
        }
      grp_sync(g);
      if (g.rank == 0 && mt > 0) {  // per-leg residuals of step q (partials stable until the next barrier)
        double wq = 0.0;
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
          if (q > hc[c]) continue;
          double s2 = 0.0;
          for (int tc = 0; tc < mt; ++tc) {
            double v = 0.0;
            for (int qq = 0; qq < g.size; ++qq)
              v += (g.size > 1 ? cl.map_shared_rank(ring, qq) : ring)[(q & 1) * 256 + tc + c * mt];
            s2 += v * v;
          }
          wq = fmax(wq, sqrt(s2) / gam / cc[c]);
        }
        worst = fmax(worst, block_max(wq, red));
      }
    }
    if (g.rank == 0 && threadIdx.x == 0) {
      a.res[e] = worst;
      int cv = (mt == 0) || (worst <= 1.0);
      a.conv[e] = cv;
      if (cv && a.kfin) a.kfin[e] = K;
    }
    grp_sync(g);
  }
}

void launch_small_hom(cudaStream_t st, const SPArgs& a, int nslots) {
  if (a.K + a.m > KSMALL_MAX) fail(1, "Krylov dimension exceeds the small-problem capacity");
  if (a.m > 16) fail(1, "grouped legs: at most 16 legs per group");
  ProfScope ps(PC_SMALLHOM, st, 0.0, eact(a.E, a.active) * (22.0 * a.K * a.K * a.K));
  const int ncl = std::min(a.E, nslots);
  launch_clustered(k_small_hom, ncl, cluster_size_for(ncl), HOM_DYN, st, a);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- batched expm (stage API)
__global__ void __launch_bounds__(PEXP_THREADS, SMALL_MINB)
k_expm_batched(int E, int N, const double* A, double* X, double* work, long long work_slot, int* iwork) {
  __shared__ double red[32];
  extern __shared__ double xsm[];  // HOM_DYN bytes: LU panel / permutation scratch
  const Grp g = this_grp();
  const int slot = blockIdx.x / g.size, nslot = gridDim.x / g.size;
  for (int e = slot; e < E; e += nslot) {
    double* Xe = X + size_t(e) * N * N;
    const double* Ae = A + size_t(e) * N * N;
    for (int t = threadIdx.x + g.rank * blockDim.x; t < N * N; t += blockDim.x * g.size) Xe[t] = Ae[t];
    grp_sync(g);
    cta_expm_pade13(N, Xe, N, work + slot * work_slot, N, iwork + slot * N, red, g, xsm, int(HOM_DYN / 8));
  }
}

// ---------------------------------------------------------------- host wrappers
void launch_sym_eig_select(cudaStream_t st, int E, int s, const double* G, double* lam, double* Msel,
                           int* off, double* sigma1, int pass, double tau, double theta, const int* active) {
  ProfScope ps(PC_SVDSMALL, st, 0.0, 0.0);
  k_sym_eig_select<<<E, EIG_THREADS, SM2, st>>>(s, G, lam, Msel, off, sigma1, pass, tau, theta, active);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_block_chol(cudaStream_t st, int E, int N, const double* G, long long gs_e, int ldg,
                       const double* norm0, long long ns_e, int ldn, double defl, double* Rinv, const double* Rprev,
                       long long rps_e, int ldrp, double* Rout, long long rs_e, int ldr, int* live,
                       long long ls_e, const int* active, bool pivoted, double dtol, double* norm0_out, int* maskB,
                       int* maskC) {
  if (N > MAXS) fail(1, "block width > 64 not supported");
  ProfScope ps(PC_SVDSMALL, st, 0.0, 0.0);
  k_block_chol<<<E, PEXP_THREADS, SM2, st>>>(N, G, gs_e, ldg, norm0, ns_e, ldn, defl, Rinv, Rprev, rps_e, ldrp,
                                            Rout, rs_e, ldr, live, ls_e, active, pivoted ? 1 : 0, g_cfg.piv_tol, dtol,
                                            norm0_out, maskB, maskC);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_onesided_svd(cudaStream_t st, int E, int s, const double* C, const int* kk, double tau,
                         double* Qs, double* sig, double* Cs, int* m_out, const int* active) {
  ProfScope ps(PC_SVDSMALL, st, 0.0, 0.0);
  k_onesided_svd<<<E, PEXP_THREADS, SM2, st>>>(s, C, kk, tau, Qs, sig, Cs, m_out, active);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_build_final(cudaStream_t st, int E, int s, int mmax, const int* kk, const double* Qs,
                        const double* sig, const double* Cs, const int* m, double* Msel, double* Cfin,
                        int* fill) {
  ProfScope ps(PC_SVDSMALL, st, 0.0, 0.0);
  k_build_final<<<E, PEXP_THREADS, 0, st>>>(s, mmax, kk, Qs, sig, Cs, m, Msel, Cfin, fill);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_spline(cudaStream_t st, int E, int s, int mmax, const double* Kinv, const double* Cfin,
                   double h, double eta, double* coef, double* crit) {
  size_t smem = size_t(3) * mmax * s * sizeof(double);
  ProfScope ps(PC_SVDSMALL, st, 0.0, 0.0);
  k_spline<<<E, PEXP_THREADS, smem, st>>>(s, mmax, Kinv, Cfin, h, eta, coef, crit, nullptr);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_poly_coef(cudaStream_t st, int E, int s, int mmax, int nq, const double* Dmat, const double* Cfin,
                      double eta, double* coef, double* crit) {
  ProfScope ps(PC_SVDSMALL, st, 0.0, 0.0);
  k_poly_coef<<<E, PEXP_THREADS, size_t(mmax) * s * sizeof(double), st>>>(s, mmax, nq, Dmat, Cfin, eta, coef, crit);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_small_problem(cudaStream_t st, const SPArgs& a, int nslots, int Dmax) {
  if (Dmax + a.K + a.m > KSMALL_MAX) fail(1, "Krylov dimension exceeds the small-problem capacity");
  size_t smem = SP_DYN;
  {
  const double N = Dmax + a.K + (a.kind == 0 ? double(a.nq) * a.m : 0.0);
  ProfScope ps(PC_SMALL, st, 0.0, eact(a.E, a.active) * (22.0 * N * N * N + 2.0 * a.K * a.K * a.K));
  const int ncl = std::min(a.E, nslots);
  launch_clustered(k_small_problem, ncl, cluster_size_for(ncl), smem, st, a);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_expm_batched(cudaStream_t st, int E, int N, const double* A, double* X, double* work,
                         long long work_slot, int* iwork, int nslots) {
  const int ncl = std::min(E, nslots);
  launch_clustered(k_expm_batched, ncl, cluster_size_for(ncl), HOM_DYN, st, E, N, A, X, work, work_slot, iwork);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void small_init() {
  cudaFuncSetAttribute(k_small_problem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_small_hom, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_expm_batched, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_sym_eig_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM2);
  cudaFuncSetAttribute(k_block_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM2);
  cudaFuncSetAttribute(k_onesided_svd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM2);
  cudaFuncSetAttribute(k_small_problem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SP_DYN);
  cudaFuncSetAttribute(k_small_hom, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HOM_DYN);
  cudaFuncSetAttribute(k_expm_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HOM_DYN);
  cudaFuncSetAttribute(k_spline, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 64 * 64 * 8);
}

}  // namespace pexp
