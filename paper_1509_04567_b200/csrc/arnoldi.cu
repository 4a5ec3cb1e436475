// arnoldi.cu — fused shift-and-invert block Arnoldi step (subsystems 1 + 2), one CTA per
// evaluation.  One launch performs, for every active evaluation e:
//   W0 = (I - gamma A_e)^{-1} V_b                       (two affine-scan passes per column)
//   H[0:nv, b] = V^T W0 ;  W = W0 - V H                 (BCGS pass 1: V streamed twice)
//   in-block QR: pivoted Cholesky-QR accepting well-separated columns, deferred columns
//                re-orthogonalised explicitly (CGS2), final pivoted Cholesky-QR with deflation
//   pass 2: T = V^T W ; W -= V T ; Cholesky-QR           (V streamed twice)
//   H[nv:nv+m, b] = Q^T W0                               (exact subdiagonal block)
// The new block and all small matrices live in shared memory chunks; V is read four times per
// step straight from L2/HBM with coalesced 256-B warp loads.  This replaces ~25 small kernel
// launches per step of the multi-kernel route (kept for very small batches, e.g. the Burgers scan).
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace pexp {

struct SmemT {
  double *Hs, *Cx, *Cy, *G, *Rinv, *Mc, *S, *Xw, *Lp, *d, *n0, *n0p;
  int ldc;  // chunk leading dimension (rc + 1)
};

// H_s[a + b*ldh] = sum_r V[a][r] W[b][r], a < nv, b < m
template <int MB>
__device__ inline void cta_vtw(int n, const double* V, int nv, const double* W, int m, double* Hs, int ldh, double* Cb,
                               int rc, int ldc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = PEXP_THREADS / 32;
  for (int i = threadIdx.x; i < nv * m; i += PEXP_THREADS) Hs[(i % nv) + size_t(i / nv) * ldh] = 0.0;
  for (int r0 = 0; r0 < n; r0 += rc) {
    const int rows = min(rc, n - r0);
    __syncthreads();
    for (int i = threadIdx.x; i < m * rc; i += PEXP_THREADS) {
      int bb = i / rc, r = i % rc;
      Cb[bb * ldc + r] = r < rows ? W[size_t(bb) * n + r0 + r] : 0.0;
    }
    __syncthreads();
    for (int a = warp; a < nv; a += nw) {
      const double* vc = V + size_t(a) * n + r0;
      double acc[MB];
#pragma unroll
      for (int bb = 0; bb < MB; ++bb) acc[bb] = 0.0;
      int r = lane;
      constexpr int U = 16;  // independent 256-B warp loads in flight per lane
      for (; r + 32 * (U - 1) < rows; r += 32 * U) {
        double x[U];
#pragma unroll
        for (int q = 0; q < U; ++q) x[q] = __ldcg(vc + r + 32 * q);
#pragma unroll
        for (int bb = 0; bb < MB; ++bb)
          if (bb < m) {
            const double* c = Cb + bb * ldc + r;
#pragma unroll
            for (int q = 0; q < U; ++q) acc[bb] = fma(x[q], c[32 * q], acc[bb]);
          }
      }
      for (; r < rows; r += 32) {
        double x0 = vc[r];
#pragma unroll
        for (int bb = 0; bb < MB; ++bb)
          if (bb < m) acc[bb] = fma(x0, Cb[bb * ldc + r], acc[bb]);
      }
#pragma unroll
      for (int bb = 0; bb < MB; ++bb)
        if (bb < m) {
          double v = warp_sum(acc[bb]);
          if (lane == 0) Hs[a + size_t(bb) * ldh] += v;  // column a owned by this warp
        }
    }
  }
  __syncthreads();
}

// W[b][r] -= sum_a V[a][r] Hs[a + b*ldh]
template <int MB>
__device__ inline void cta_update(int n, const double* V, int nv, double* W, int m, const double* Hs, int ldh) {
  constexpr int RR = 2, UA = 8;  // rows per thread x columns in flight
  for (int r0 = threadIdx.x; r0 < n; r0 += PEXP_THREADS * RR) {
    double acc[RR][MB];
#pragma unroll
    for (int q = 0; q < RR; ++q)
#pragma unroll
      for (int bb = 0; bb < MB; ++bb) acc[q][bb] = 0.0;
    const bool ok1 = r0 + PEXP_THREADS < n;
    int a = 0;
    for (; a + UA - 1 < nv; a += UA) {
      double x[UA][RR];
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        x[u][0] = __ldcg(V + size_t(a + u) * n + r0);
        x[u][1] = ok1 ? __ldcg(V + size_t(a + u) * n + r0 + PEXP_THREADS) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UA; ++u)
#pragma unroll
        for (int bb = 0; bb < MB; ++bb)
          if (bb < m) {
            const double h = Hs[a + u + size_t(bb) * ldh];
            acc[0][bb] = fma(x[u][0], h, acc[0][bb]);
            acc[1][bb] = fma(x[u][1], h, acc[1][bb]);
          }
    }
    for (; a < nv; ++a) {
      double x0 = V[size_t(a) * n + r0], x1 = ok1 ? V[size_t(a) * n + r0 + PEXP_THREADS] : 0.0;
#pragma unroll
      for (int bb = 0; bb < MB; ++bb)
        if (bb < m) {
          const double h = Hs[a + size_t(bb) * ldh];
          acc[0][bb] = fma(x0, h, acc[0][bb]);
          acc[1][bb] = fma(x1, h, acc[1][bb]);
        }
    }
#pragma unroll
    for (int bb = 0; bb < MB; ++bb)
      if (bb < m) {
        W[size_t(bb) * n + r0] -= acc[0][bb];
        if (ok1) W[size_t(bb) * n + r0 + PEXP_THREADS] -= acc[1][bb];
      }
  }
  __syncthreads();
}

// G[a + b*MB] = sum_r X[a][r] Y[b][r]  (Y may equal X): (column a, column-pair group) owned by a
// warp, lanes stride the rows (coalesced loads from L2), shuffle reduction.
template <int MB>
__device__ inline void cta_gram(int n, const double* X, const double* Y, int m, double* G, double*, double*, int,
                                int) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = PEXP_THREADS / 32;
  for (int a = warp; a < m; a += nw) {
    const double* xa = X + size_t(a) * n;
    double acc[MB];
#pragma unroll
    for (int bb = 0; bb < MB; ++bb) acc[bb] = 0.0;
    for (int r = lane; r < n; r += 32) {
      const double xv = __ldcg(xa + r);
#pragma unroll
      for (int bb = 0; bb < MB; ++bb)
        if (bb < m) acc[bb] = fma(xv, __ldcg(Y + size_t(bb) * n + r), acc[bb]);
    }
#pragma unroll
    for (int bb = 0; bb < MB; ++bb)
      if (bb < m) {
        double v = warp_sum(acc[bb]);
        if (lane == 0) G[a + bb * MB] = v;
      }
  }
  __syncthreads();
}

// W <- beta*W + W*M  (M: m x m, ld MB) row by row
template <int MB>
__device__ inline void cta_apply(int n, double* W, int m, const double* M, double beta) {
  for (int r = threadIdx.x; r < n; r += PEXP_THREADS) {
    double w[MB], o[MB];
#pragma unroll
    for (int bb = 0; bb < MB; ++bb) w[bb] = bb < m ? W[size_t(bb) * n + r] : 0.0;
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      double v = beta * w[c];
#pragma unroll
      for (int bb = 0; bb < MB; ++bb) v = fma(w[bb], M[bb + c * MB], v);
      o[c] = v;
    }
#pragma unroll
    for (int c = 0; c < MB; ++c)
      if (c < m) W[size_t(c) * n + r] = o[c];
  }
  __syncthreads();
}

// Pivoted, diagonally scaled, deflating Cholesky of the Gram G (m x m, ld MB) -> Rinv (ld MB),
// classes cls (1 accepted, 2 deferred, 0 dead), optional re-ordered norm0 (see k_block_chol).
template <int MB>
__device__ inline void cta_chol_piv(int m, const double* G, const double* norm0, double defl, double dtol,
                                    double piv_tol, SmemT& s, int* cls, int* perm, int* used, int* dead) {
  constexpr int LD = MB + 1;
  __shared__ int s_np, s_j, s_nd;
  __shared__ double s_piv;
  for (int k = threadIdx.x; k < m; k += PEXP_THREADS) {
    double g = G[k + k * MB];
    bool dk = !(g > 0.0);
    if (norm0 && !(g > defl * defl * norm0[k])) dk = true;
    dead[k] = dk;
    used[k] = 0;
    s.d[k] = g > 0.0 ? 1.0 / sqrt(g) : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < m * m; idx += PEXP_THREADS) {
    int i = idx % m, j = idx / m;
    s.S[i * LD + j] = s.d[i] * s.d[j] * 0.5 * (G[i + j * MB] + G[j + i * MB]);
    s.Lp[i * LD + j] = 0.0;
  }
  if (threadIdx.x == 0) s_np = 0;
  __syncthreads();
  for (int t = 0; t < m; ++t) {
    if (threadIdx.x == 0) {
      int jb = -1;
      double best = dtol > 0.0 ? dtol : piv_tol;
      for (int j = 0; j < m; ++j)
        if (!used[j] && !dead[j] && s.S[j * LD + j] > best) { best = s.S[j * LD + j]; jb = j; }
      s_j = jb;
      if (jb >= 0) {
        used[jb] = 1;
        perm[t] = jb;
        s_piv = sqrt(best);
        s_np = t + 1;
      }
    }
    __syncthreads();
    const int jb = s_j;
    if (jb < 0) break;
    const double pv = s_piv;
    for (int i = threadIdx.x; i < m; i += PEXP_THREADS)
      s.Xw[i * LD] = (i == jb) ? pv : (used[i] ? 0.0 : s.S[i * LD + jb] / pv);
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * m; idx += PEXP_THREADS) {
      int i = idx % m, k = idx / m;
      if (!used[i] && !used[k]) s.S[i * LD + k] -= s.Xw[i * LD] * s.Xw[k * LD];
    }
    for (int i = threadIdx.x; i < m; i += PEXP_THREADS) s.Lp[i * LD + t] = s.Xw[i * LD];
    __syncthreads();
  }
  const int np = s_np;
  if (threadIdx.x == 0) {
    int q = np, nd = 0;
    if (dtol > 0.0)
      for (int j = 0; j < m; ++j)
        if (!used[j] && !dead[j]) { perm[q++] = j; ++nd; }
    for (int j = 0; j < m; ++j)
      if (!used[j] && (dtol <= 0.0 || dead[j])) perm[q++] = j;
    s_nd = nd;
  }
  __syncthreads();
  const int nd = s_nd;
  // X = Rp^{-1} (leading np x np), Rp[t][a] = Lp[perm[a]][t]
  for (int j = threadIdx.x; j < m; j += PEXP_THREADS) {
    for (int k = 0; k < m; ++k) s.Xw[k * LD + j] = 0.0;
    if (j < np)
      for (int k = j; k >= 0; --k) {
        double sum = (k == j) ? 1.0 : 0.0;
        for (int q = k + 1; q <= j; ++q) sum -= s.Lp[perm[q] * LD + k] * s.Xw[q * LD + j];
        s.Xw[k * LD + j] = sum / s.Lp[perm[k] * LD + k];
      }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < MB * MB; idx += PEXP_THREADS) s.Rinv[idx] = 0.0;
  __syncthreads();
  for (int idx = threadIdx.x; idx < m * m; idx += PEXP_THREADS) {
    int a = idx % m, t = idx / m;
    s.Rinv[perm[a] + t * MB] = s.d[perm[a]] * s.Xw[a * LD + t];
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nd; q += PEXP_THREADS) s.Rinv[perm[np + q] + (np + q) * MB] = 1.0;
  for (int k = threadIdx.x; k < m; k += PEXP_THREADS) {
    cls[k] = k < np ? 1 : (k < np + nd ? 2 : 0);
    if (norm0) s.n0p[k] = norm0[perm[k]];
  }
  __syncthreads();
}

template <int MB>
__global__ void __launch_bounds__(PEXP_THREADS) k_arnoldi_step(StepArgs A) {
  extern __shared__ double sm[];
  __shared__ Aff wsm[PEXP_THREADS / 32 + 1];
  __shared__ double red[32];
  __shared__ int cls[MB], perm[MB], used[MB], dead[MB];
  const int e = blockIdx.x;
  if (A.active && !A.active[e]) return;
  const int n = A.n, m = A.m, b = A.b, kcap = A.kcap, nv = (b + 1) * m, rc = A.rc;
  SmemT s;
  s.ldc = rc + 1;
  const int cbuf = max(s.ldc * MB, PEXP_THREADS * SPAD);
  double* p = sm;
  s.Hs = p; p += size_t(kcap) * MB;
  s.Cx = p; p += cbuf;
  s.Cy = p; p += cbuf;
  s.G = p; p += MB * MB;
  s.Rinv = p; p += MB * MB;
  s.Mc = p; p += MB * MB;
  s.S = p; p += MB * (MB + 1);
  s.Xw = p; p += MB * (MB + 1);
  s.Lp = p; p += MB * (MB + 1);
  s.d = p; p += MB;
  s.n0 = p; p += MB;
  s.n0p = p; p += MB;
  double* V = A.V + e * A.vs_e;
  double* H = A.H + e * A.hs_e;
  int* live = A.live + size_t(e) * kcap;
  double* W0 = A.W0 + e * A.w0s_e;
  double* W = V + size_t(nv) * n;
  const size_t fo = size_t(A.fidx ? A.fidx[e] : e) * n;
  // ---- W0 = (I - gamma A)^{-1} V_b   (kept in W0; working copy in the new block)
  for (int c = 0; c < m; ++c) {
    double nr = cta_sai_solve(n, A.periodic, A.fl + fo, A.fdinv + fo, A.fsup + fo, A.periodic ? A.fz + fo : nullptr,
                              A.periodic ? A.fw + fo : nullptr, V + size_t(b * m + c) * n, W + size_t(c) * n,
                              W0 + size_t(c) * n, s.Cx, s.Cy, wsm, red);
    if (threadIdx.x == 0) s.n0[c] = nr;
  }
  __syncthreads();
  // ---- BCGS pass 1
  cta_vtw<MB>(n, V, nv, W, m, s.Hs, kcap, s.Cx, rc, s.ldc);
  for (int i = threadIdx.x; i < nv * m; i += PEXP_THREADS) {
    int a = i % nv, c = i / nv;
    H[a + size_t(b * m + c) * kcap] = s.Hs[a + size_t(c) * kcap];
  }
  cta_update<MB>(n, V, nv, W, m, s.Hs, kcap);
  // ---- in-block QR, stage A (accept kappa <= 1e4, defer the rest, drop below defl*|W0|)
  cta_gram<MB>(n, W, W, m, s.G, s.Cx, s.Cy, rc, s.ldc);
  cta_chol_piv<MB>(m, s.G, s.n0, A.defl, 1e-8, A.piv_tol, s, cls, perm, used, dead);
  cta_apply<MB>(n, W, m, s.Rinv, 0.0);
  // ---- stage B: explicit CGS2 of deferred columns against accepted ones
  for (int rep = 0; rep < 2; ++rep) {
    cta_gram<MB>(n, W, W, m, s.G, s.Cx, s.Cy, rc, s.ldc);
    for (int idx = threadIdx.x; idx < MB * MB; idx += PEXP_THREADS) {
      int a = idx % MB, k = idx / MB;
      s.Mc[idx] = (a < m && k < m && cls[a] == 1 && cls[k] == 2) ? -s.G[a + k * MB] : 0.0;
    }
    __syncthreads();
    cta_apply<MB>(n, W, m, s.Mc, 1.0);
  }
  // ---- stage C: final pivoted CholQR with deflation relative to |W0|
  cta_gram<MB>(n, W, W, m, s.G, s.Cx, s.Cy, rc, s.ldc);
  for (int k = threadIdx.x; k < m; k += PEXP_THREADS) s.n0[k] = s.n0p[k];
  __syncthreads();
  cta_chol_piv<MB>(m, s.G, s.n0, A.defl, 0.0, A.piv_tol, s, cls, perm, used, dead);
  cta_apply<MB>(n, W, m, s.Rinv, 0.0);
  // ---- BCGS pass 2 + CholQR
  cta_vtw<MB>(n, V, nv, W, m, s.Hs, kcap, s.Cx, rc, s.ldc);
  cta_update<MB>(n, V, nv, W, m, s.Hs, kcap);
  cta_gram<MB>(n, W, W, m, s.G, s.Cx, s.Cy, rc, s.ldc);
  cta_chol_piv<MB>(m, s.G, nullptr, A.defl, 0.0, A.piv_tol, s, cls, perm, used, dead);
  cta_apply<MB>(n, W, m, s.Rinv, 0.0);
  // ---- subdiagonal block H[nv + a, b*m + c] = Q_a^T W0_c ; live flags
  cta_gram<MB>(n, W, W0, m, s.G, s.Cx, s.Cy, rc, s.ldc);
  for (int i = threadIdx.x; i < m * m; i += PEXP_THREADS) {
    int a = i % m, c = i / m;
    H[nv + a + size_t(b * m + c) * kcap] = s.G[a + c * MB];
  }
  for (int k = threadIdx.x; k < m; k += PEXP_THREADS) live[nv + k] = cls[k] ? 1 : 0;
}

static size_t step_smem(int MB, int kcap, int rc) {
  int ldc = rc + 1;
  size_t cbuf = std::max(size_t(ldc) * MB, size_t(PEXP_THREADS) * SPAD);
  return sizeof(double) * (size_t(kcap) * MB + 2 * cbuf + 3 * MB * MB + 3 * MB * (MB + 1) + 3 * MB);
}

int step_rc(int MB) { return MB <= 8 ? 512 : (MB <= 16 ? 256 : 128); }

bool arnoldi_fused_ok(int m, int kcap) {
  if (m > 32) return false;
  int MB = m <= 8 ? 8 : (m <= 16 ? 16 : 32);
  return step_smem(MB, kcap, step_rc(MB)) <= 220 * 1024;
}

extern double g_piv_tol;

void launch_arnoldi_step(cudaStream_t st, StepArgs a) {
  const int MB = a.m <= 8 ? 8 : (a.m <= 16 ? 16 : 32);
  a.rc = step_rc(MB);
  a.piv_tol = g_piv_tol;
  size_t smem = step_smem(MB, a.kcap, a.rc);
  const int nv = (a.b + 1) * a.m;
  ProfScope ps(PC_ARNOLDI, st, double(a.E) * a.n * 8.0 * (4.0 * nv + 12.0 * a.m),
               double(a.E) * a.n * (8.0 * nv * a.m + 10.0 * a.m * a.m));
  if (MB == 8) {
    cudaFuncSetAttribute(k_arnoldi_step<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_arnoldi_step<8><<<a.E, PEXP_THREADS, smem, st>>>(a);
  } else if (MB == 16) {
    cudaFuncSetAttribute(k_arnoldi_step<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_arnoldi_step<16><<<a.E, PEXP_THREADS, smem, st>>>(a);
  } else {
    cudaFuncSetAttribute(k_arnoldi_step<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_arnoldi_step<32><<<a.E, PEXP_THREADS, smem, st>>>(a);
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
}

}  // namespace pexp
