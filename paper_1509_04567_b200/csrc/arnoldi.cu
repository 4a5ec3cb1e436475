// arnoldi.cu — fused shift-and-invert block Arnoldi step (subsystems 1 + 2), one thread-block
// CLUSTER per evaluation (PAPER.md:171-176 Eq.(blockKrylovSubspace), SaI P:176).  One launch
// performs, for every active evaluation e:
//   W0 = (I - gamma A_e)^{-1} V_b                       (affine-scan passes, carries across the cluster)
//   H[0:nv, b] = V^T W0 ;  W = W0 - V H                 (BCGS pass 1: V streamed twice)
//   in-block QR: pivoted Cholesky-QR accepting well-separated columns, deferred columns
//                re-orthogonalised explicitly (CGS2), final pivoted Cholesky-QR with deflation
//   pass 2: T = V^T W ; W -= V T ; Cholesky-QR           (V streamed twice)
//   H[nv:nv+m, b] = Q^T W0                               (exact subdiagonal block)
// The rows of every column are split over the cs CTAs of the cluster.  Every reduction over
// rows (V^T W, the block Grams, the solve's carries and norms) is a per-CTA partial in shared
// memory summed over the cluster through distributed shared memory in rank order, so all CTAs
// hold bitwise identical small matrices and take identical pivoting/deflation decisions (the
// small m x m Cholesky work is simply repeated per CTA).  V is read four times per step straight
// from L2/HBM with coalesced 256-B warp loads.  This replaces ~25 small kernel launches per step
// of the multi-kernel route (kept for steps whose panels do not fit shared memory).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

namespace pexp {

struct SmemT {
  double *Hs, *Pp, *Cx, *Cy, *G, *Gp, *Rinv, *Mc, *S, *Xw, *Lp, *d, *n0, *n0p, *xch, *Ws;
  int ldc;   // chunk leading dimension (rc + 1)
  int gpar;  // which of the two Gram partial buffers the next cluster reduction uses
};

constexpr int RC = 256;  // rows per staged chunk of the projections (8 rows per lane)

// rows of every column owned by one CTA of a cs-CTA cluster (multiple of 32)
__host__ __device__ inline int step_rows(int n, int cs) { return ((n + cs - 1) / cs + 31) / 32 * 32; }

__device__ inline void cl_sync(cg::cluster_group& cl, int cs) {
  if (cs > 1)
    cl.sync();
  else
    __syncthreads();
}

// Cluster sum of per-CTA partials kept in GLOBAL memory: rank q's partial at part0 + q * stride.
__device__ inline void cl_allreduce_g(cg::cluster_group& cl, int cs, const double* part0, long long stride,
                                      double* out, int cnt) {
  cl_sync(cl, cs);
  for (int i = threadIdx.x; i < cnt; i += PEXP_THREADS) {
    double s = 0.0;
    for (int q = 0; q < cs; ++q) s += __ldcg(part0 + q * stride + i);
    out[i] = s;
  }
  __syncthreads();
}

// out[i] = sum over the cluster's CTAs (rank order) of part[i], i < cnt.  part and out distinct.
// One cluster barrier: a CTA may overwrite `part` only after the NEXT cluster barrier (all remote
// reads of this reduction happen before their reader arrives there), so consecutive reductions
// alternate buffers (Gram partials) or are separated by other reductions (V^T W partials).
__device__ inline void cl_allreduce(cg::cluster_group& cl, int cs, double* part, double* out, int cnt) {
  cl_sync(cl, cs);
  for (int i = threadIdx.x; i < cnt; i += PEXP_THREADS) {
    double s = 0.0;
    for (int q = 0; q < cs; ++q) s += (cs > 1 ? cl.map_shared_rank(part, q) : part)[i];
    out[i] = s;
  }
  __syncthreads();
}

// Partial Hp[a + c*nv] = sum over this CTA's rows of V[a][r] W[c][r]  (a < nv, c < m).
// The W chunk (RC rows) is staged in shared memory; every warp streams two V columns at a time
// (16 independent 256-B loads in flight per lane) and reduces with shuffles.
template <int MB>
__device__ inline void cta_vtw(int ld, int ldw, int rows, const double* V, int nv, const double* W, int m,
                               double* Hp, double* Cb, int ldc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = PEXP_THREADS / 32;
  constexpr int U = RC / 32;
  for (int i = threadIdx.x; i < nv * m; i += PEXP_THREADS) Hp[i] = 0.0;
  constexpr int CPW = MB <= 16 ? 2 : 1;  // columns per warp pass (register budget)
  for (int r0 = 0; r0 < rows; r0 += RC) {
    const int cnt = min(RC, rows - r0);
    __syncthreads();
    for (int i = threadIdx.x; i < m * RC; i += PEXP_THREADS) {
      int bb = i / RC, r = i % RC;
      Cb[bb * ldc + r] = r < cnt ? W[size_t(bb) * ldw + r0 + r] : 0.0;
    }
    __syncthreads();
    for (int a = CPW * warp; a < nv; a += CPW * nw) {
      const bool two = CPW == 2 && a + 1 < nv;
      const double* v0 = V + size_t(a) * ld + r0;
      const double* v1 = V + size_t(a + 1) * ld + r0;
      double x0[U], x1[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int r = lane + 32 * q;
        x0[q] = r < cnt ? __ldcg(v0 + r) : 0.0;
        x1[q] = (two && r < cnt) ? __ldcg(v1 + r) : 0.0;
      }
      double acc0[MB], acc1[MB];
#pragma unroll
      for (int bb = 0; bb < MB; ++bb) { acc0[bb] = 0.0; acc1[bb] = 0.0; }
#pragma unroll
      for (int bb = 0; bb < MB; ++bb)
        if (bb < m) {
          const double* c = Cb + bb * ldc + lane;
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const double cv = c[32 * q];
            acc0[bb] = fma(x0[q], cv, acc0[bb]);
            acc1[bb] = fma(x1[q], cv, acc1[bb]);
          }
        }
#pragma unroll
      for (int bb = 0; bb < MB; ++bb)
        if (bb < m) {
          const double s0 = warp_sum(acc0[bb]);
          const double s1 = warp_sum(acc1[bb]);
          if (lane == 0) {  // columns a, a+1 owned by this warp: no race
            Hp[a + bb * nv] += s0;
            if (two) Hp[a + 1 + bb * nv] += s1;
          }
        }
    }
  }
  __syncthreads();
}

// W[b][r] -= sum_a V[a][r] Hs[a + b*nv] on this CTA's rows
template <int MB>
__device__ inline void cta_update(int ld, int ldw, int rows, const double* V, int nv, double* W, int m,
                                  const double* Hs) {
  constexpr int RR = 2, UA = 8;  // rows per thread x columns in flight
  for (int r0 = threadIdx.x; r0 < rows; r0 += PEXP_THREADS * RR) {
    double acc[RR][MB];
#pragma unroll
    for (int q = 0; q < RR; ++q)
#pragma unroll
      for (int bb = 0; bb < MB; ++bb) acc[q][bb] = 0.0;
    const bool ok1 = r0 + PEXP_THREADS < rows;
    int a = 0;
    for (; a + UA - 1 < nv; a += UA) {
      double x[UA][RR];
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        x[u][0] = __ldcg(V + size_t(a + u) * ld + r0);
        x[u][1] = ok1 ? __ldcg(V + size_t(a + u) * ld + r0 + PEXP_THREADS) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UA; ++u)
#pragma unroll
        for (int bb = 0; bb < MB; ++bb)
          if (bb < m) {
            const double h = Hs[a + u + bb * nv];
            acc[0][bb] = fma(x[u][0], h, acc[0][bb]);
            acc[1][bb] = fma(x[u][1], h, acc[1][bb]);
          }
    }
    for (; a < nv; ++a) {
      double x0 = V[size_t(a) * ld + r0], x1 = ok1 ? V[size_t(a) * ld + r0 + PEXP_THREADS] : 0.0;
#pragma unroll
      for (int bb = 0; bb < MB; ++bb)
        if (bb < m) {
          const double h = Hs[a + bb * nv];
          acc[0][bb] = fma(x0, h, acc[0][bb]);
          acc[1][bb] = fma(x1, h, acc[1][bb]);
        }
    }
#pragma unroll
    for (int bb = 0; bb < MB; ++bb)
      if (bb < m) {
        W[size_t(bb) * ldw + r0] -= acc[0][bb];
        if (ok1) W[size_t(bb) * ldw + r0 + PEXP_THREADS] -= acc[1][bb];
      }
  }
  __syncthreads();
}

// Partial G[a + b*MB] = sum over this CTA's rows of X[a][r] Y[b][r]  (Y may equal X)
template <int MB>
__device__ inline void cta_gram(int ldx, int ldy, int rows, const double* X, const double* Y, int m, double* G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = PEXP_THREADS / 32;
  for (int a = warp; a < m; a += nw) {
    const double* xa = X + size_t(a) * ldx;
    double acc[MB];
#pragma unroll
    for (int bb = 0; bb < MB; ++bb) acc[bb] = 0.0;
    for (int r = lane; r < rows; r += 32) {
      const double xv = xa[r];
#pragma unroll
      for (int bb = 0; bb < MB; ++bb)
        if (bb < m) acc[bb] = fma(xv, Y[size_t(bb) * ldy + r], acc[bb]);
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

// Cluster-wide Gram: partial into s.Gp, summed into s.G
template <int MB>
__device__ inline void cl_gram(cg::cluster_group& cl, int cs, int ldx, int ldy, int rows, const double* X,
                               const double* Y, int m, SmemT& s) {
  double* gp = s.Gp + s.gpar * MB * MB;
  s.gpar ^= 1;
  for (int i = threadIdx.x; i < MB * MB; i += PEXP_THREADS) gp[i] = 0.0;
  __syncthreads();
  cta_gram<MB>(ldx, ldy, rows, X, Y, m, gp);
  cl_allreduce(cl, cs, gp, s.G, MB * MB);
}

// W <- beta*W + W*M  (M: m x m, ld MB) row by row
template <int MB>
__device__ inline void cta_apply(int ld, int rows, double* W, int m, const double* M, double beta) {
  for (int r = threadIdx.x; r < rows; r += PEXP_THREADS) {
    double w[MB], o[MB];
#pragma unroll
    for (int bb = 0; bb < MB; ++bb) w[bb] = bb < m ? W[size_t(bb) * ld + r] : 0.0;
#pragma unroll
    for (int c = 0; c < MB; ++c) {
      double v = beta * w[c];
#pragma unroll
      for (int bb = 0; bb < MB; ++bb) v = fma(w[bb], M[bb + c * MB], v);
      o[c] = v;
    }
#pragma unroll
    for (int c = 0; c < MB; ++c)
      if (c < m) W[size_t(c) * ld + r] = o[c];
  }
  __syncthreads();
}

// Pivoted, diagonally scaled, deflating Cholesky of the Gram G (m x m, ld MB) -> Rinv (ld MB),
// classes cls (1 accepted, 2 deferred, 0 dead), optional re-ordered norm0 (see k_block_chol).
// m <= 32: the whole factorisation runs in warp 0 (lane i owns row i; warp argmax for the pivot,
// __syncwarp between phases, no CTA barriers); one __syncthreads publishes the results.
// Returns the smallest accepted scaled pivot (squared), +inf if none was accepted.
template <int MB>
__device__ inline double cta_chol_piv(int m, const double* G, const double* norm0, double defl, double dtol,
                                      double piv_tol, SmemT& s, int* cls, int* perm, int* used, int* dead) {
  constexpr int LD = MB + 1;
  __shared__ double s_pmin;
  if (threadIdx.x < 32) {
    const int i = threadIdx.x;
    const unsigned full = 0xffffffffu;
    if (i < m) {
      const double g = G[i + i * MB];
      bool di = !(g > 0.0);
      if (norm0 && !(g > defl * defl * norm0[i])) di = true;
      dead[i] = di;
      used[i] = 0;
      s.d[i] = g > 0.0 ? 1.0 / sqrt(g) : 0.0;
    }
    __syncwarp();
    if (i < m)
      for (int j = 0; j < m; ++j) {
        s.S[i * LD + j] = s.d[i] * s.d[j] * 0.5 * (G[i + j * MB] + G[j + i * MB]);
        s.Lp[i * LD + j] = 0.0;
      }
    __syncwarp();
    const double best0 = dtol > 0.0 ? dtol : piv_tol;
    int np = 0;
    double pmin = INFINITY;
    for (int t = 0; t < m; ++t) {
      // argmax of the remaining scaled pivots (strictly above best0; ties -> lowest index)
      double cv = -1.0;
      if (i < m && !used[i] && !dead[i] && s.S[i * LD + i] > best0) cv = s.S[i * LD + i];
      int ci = i;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(full, cv, o);
        const int oi = __shfl_xor_sync(full, ci, o);
        if (ov > cv || (ov == cv && oi < ci)) { cv = ov; ci = oi; }
      }
      if (cv < 0.0) break;  // uniform over the warp
      pmin = fmin(pmin, cv);
      const int jb = ci;
      const double pv = sqrt(cv);
      double xw = 0.0;
      if (i < m) xw = (i == jb) ? pv : (used[i] ? 0.0 : s.S[i * LD + jb] / pv);
      __syncwarp();
      if (i == 0) { used[jb] = 1; perm[t] = jb; }
      __syncwarp();
      if (i < m) {
        s.Xw[i * LD] = xw;
        s.Lp[i * LD + t] = xw;
      }
      __syncwarp();
      if (i < m && !used[i])
        for (int k = 0; k < m; ++k)
          if (!used[k]) s.S[i * LD + k] -= xw * s.Xw[k * LD];
      __syncwarp();
      np = t + 1;
    }
    int nd = 0;
    if (i == 0) {
      int q = np;
      if (dtol > 0.0)
        for (int j = 0; j < m; ++j)
          if (!used[j] && !dead[j]) { perm[q++] = j; ++nd; }
      for (int j = 0; j < m; ++j)
        if (!used[j] && (dtol <= 0.0 || dead[j])) perm[q++] = j;
    }
    nd = __shfl_sync(full, nd, 0);
    __syncwarp();
    // X = Rp^{-1} (leading np x np), Rp[t][a] = Lp[perm[a]][t]; lane j owns column j
    if (i < m) {
      for (int k = 0; k < m; ++k) s.Xw[k * LD + i] = 0.0;
      if (i < np)
        for (int k = i; k >= 0; --k) {
          double sum = (k == i) ? 1.0 : 0.0;
          for (int q = k + 1; q <= i; ++q) sum -= s.Lp[perm[q] * LD + k] * s.Xw[q * LD + i];
          s.Xw[k * LD + i] = sum / s.Lp[perm[k] * LD + k];
        }
    }
    __syncwarp();
    for (int idx = i; idx < MB * MB; idx += 32) s.Rinv[idx] = 0.0;
    __syncwarp();
    for (int idx = i; idx < m * m; idx += 32) {
      const int a = idx % m, t = idx / m;
      s.Rinv[perm[a] + t * MB] = s.d[perm[a]] * s.Xw[a * LD + t];
    }
    __syncwarp();
    if (i < nd) s.Rinv[perm[np + i] + (np + i) * MB] = 1.0;
    if (i < m) {
      cls[i] = i < np ? 1 : (i < np + nd ? 2 : 0);
      if (norm0) s.n0p[i] = norm0[perm[i]];
    }
    if (i == 0) s_pmin = pmin;
  }
  __syncthreads();
  return s_pmin;
}

// ---------------------------------------------------------------- cluster-split SaI solve
// Forward L-solve y_g = -l_g y_{g-1} + b_g and backward U-solve x_g = -d_g c_g x_{g+1} + d_g y_g
// as affine maps (scan.cuh), for a group of up to CB columns at once: the maps of all columns of
// a row share their multiplier (-l_g, resp. -d_g c_g) and differ only in the offset, so one block
// scan carries 1 + CB values.  Rows [g0, g0 + cnt) belong to this CTA; thread t composes the EPT
// consecutive rows t*EPT.. of each CHUNK; chunks are chained through the running carry.
constexpr int CB = 8;

// Exclusive block scan of (A, B[CB]) maps ordered by rank (REV: rank = 255 - threadIdx.x).
// Returns the exclusive prefix in (pA, pB) and the block total in (tA, tB).
template <bool REV>
__device__ inline void block_scan_multi(double A, const double (&B)[CB], double* wsmM, double& pA, double (&pB)[CB],
                                        double& tA, double (&tB)[CB]) {
  const int rank = REV ? PEXP_THREADS - 1 - threadIdx.x : threadIdx.x;
  const int lane = rank & 31, w = rank >> 5;
  double iA = A, iB[CB];
#pragma unroll
  for (int c = 0; c < CB; ++c) iB[c] = B[c];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double qa = REV ? __shfl_down_sync(0xffffffffu, iA, o) : __shfl_up_sync(0xffffffffu, iA, o);
    double qb[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c)
      qb[c] = REV ? __shfl_down_sync(0xffffffffu, iB[c], o) : __shfl_up_sync(0xffffffffu, iB[c], o);
    if (lane >= o) {  // (q then i): A = iA*qa, B = iA*qb + iB
#pragma unroll
      for (int c = 0; c < CB; ++c) iB[c] = fma(iA, qb[c], iB[c]);
      iA *= qa;
    }
  }
  double eA = REV ? __shfl_down_sync(0xffffffffu, iA, 1) : __shfl_up_sync(0xffffffffu, iA, 1);
  double eB[CB];
#pragma unroll
  for (int c = 0; c < CB; ++c) eB[c] = REV ? __shfl_down_sync(0xffffffffu, iB[c], 1) : __shfl_up_sync(0xffffffffu, iB[c], 1);
  if (lane == 0) {
    eA = 1.0;
#pragma unroll
    for (int c = 0; c < CB; ++c) eB[c] = 0.0;
  }
  constexpr int NW = PEXP_THREADS / 32, ST = CB + 1;
  __syncthreads();
  if (lane == 31) {
    wsmM[w * ST] = iA;
#pragma unroll
    for (int c = 0; c < CB; ++c) wsmM[w * ST + 1 + c] = iB[c];
  }
  __syncthreads();
  if (threadIdx.x < ST) {  // thread c' composes component c' over the warps (A first, then the B's)
    const int c = threadIdx.x;
    double accA = 1.0, accB = 0.0;
    for (int k = 0; k < NW; ++k) {
      const double ta = wsmM[k * ST], tb = c == 0 ? 0.0 : wsmM[k * ST + c];
      // store the exclusive prefix of warp k in slot (NW + k)
      wsmM[(NW + k) * ST + c] = c == 0 ? accA : accB;
      if (c > 0) accB = fma(ta, accB, tb);
      accA *= ta;
    }
    wsmM[2 * NW * ST + c] = c == 0 ? accA : accB;
  }
  __syncthreads();
  const double wA = wsmM[(NW + w) * ST];
  // prefix = (warp prefix) then (exclusive within the warp)
  pA = eA * wA;
#pragma unroll
  for (int c = 0; c < CB; ++c) pB[c] = fma(eA, wsmM[(NW + w) * ST + 1 + c], eB[c]);
  tA = wsmM[2 * NW * ST];
#pragma unroll
  for (int c = 0; c < CB; ++c) tB[c] = wsmM[2 * NW * ST + 1 + c];
  __syncthreads();
}

// Forward segment maps (no writes) of columns [c0, c0 + nc) of b (ld ldb): total map per column.
__device__ inline void seg_maps_fwd(int g0, int cnt, const double* l, const double* b, int ldb, int nc, double* wsmM,
                                    double& TA, double (&TB)[CB]) {
  const int t = threadIdx.x;
  TA = 1.0;
#pragma unroll
  for (int c = 0; c < CB; ++c) TB[c] = 0.0;
  for (int base = 0; base < cnt; base += CHUNK) {
    double A = 1.0, B[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) B[c] = 0.0;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = base + t * EPT + k;
      if (i < cnt) {
        const double a = -l[g0 + i];
#pragma unroll
        for (int c = 0; c < CB; ++c) B[c] = fma(a, B[c], c < nc ? b[size_t(c) * ldb + i] : 0.0);
        A *= a;
      }
    }
    double pA, pB[CB], tA, tB[CB];
    block_scan_multi<false>(A, B, wsmM, pA, pB, tA, tB);
#pragma unroll
    for (int c = 0; c < CB; ++c) TB[c] = fma(tA, TB[c], tB[c]);
    TA *= tA;
  }
}

// Forward pass with carry-in: y (ld ldy) from b (ld ldb); thread t solves its EPT rows in registers.
__device__ inline void seg_fwd_multi(int g0, int cnt, const double* l, const double* b, int ldb, double* y, int ldy,
                                     int nc, const double (&carry0)[CB], double* wsmM) {
  const int t = threadIdx.x;
  double carry[CB];
#pragma unroll
  for (int c = 0; c < CB; ++c) carry[c] = carry0[c];
  for (int base = 0; base < cnt; base += CHUNK) {
    double av[EPT], A = 1.0, B[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) B[c] = 0.0;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = base + t * EPT + k;
      av[k] = i < cnt ? -l[g0 + i] : 1.0;
      if (i < cnt) {
#pragma unroll
        for (int c = 0; c < CB; ++c) B[c] = fma(av[k], B[c], c < nc ? b[size_t(c) * ldb + i] : 0.0);
        A *= av[k];
      }
    }
    double pA, pB[CB], tA, tB[CB];
    block_scan_multi<false>(A, B, wsmM, pA, pB, tA, tB);
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      if (c < nc) {
        double v = fma(pA, carry[c], pB[c]);
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          const int i = base + t * EPT + k;
          if (i < cnt) {
            v = fma(av[k], v, b[size_t(c) * ldb + i]);
            y[size_t(c) * ldy + i] = v;
          }
        }
      }
      carry[c] = fma(tA, carry[c], tB[c]);
    }
  }
}

// Backward segment maps of y (ld ldy): total map per column (rows in descending order).
__device__ inline void seg_maps_bwd(int g0, int cnt, const double* di, const double* cs, const double* y, int ldy,
                                    int nc, double* wsmM, double& TA, double (&TB)[CB]) {
  const int t = threadIdx.x;
  TA = 1.0;
#pragma unroll
  for (int c = 0; c < CB; ++c) TB[c] = 0.0;
  for (int base = ((cnt - 1) / CHUNK) * CHUNK; base >= 0 && cnt > 0; base -= CHUNK) {
    double A = 1.0, B[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) B[c] = 0.0;
#pragma unroll
    for (int k = EPT - 1; k >= 0; --k) {
      const int i = base + t * EPT + k;
      if (i < cnt) {
        const double dv = di[g0 + i], a = -dv * cs[g0 + i];
#pragma unroll
        for (int c = 0; c < CB; ++c) B[c] = fma(a, B[c], c < nc ? dv * y[size_t(c) * ldy + i] : 0.0);
        A *= a;
      }
    }
    double pA, pB[CB], tA, tB[CB];
    block_scan_multi<true>(A, B, wsmM, pA, pB, tA, tB);
#pragma unroll
    for (int c = 0; c < CB; ++c) TB[c] = fma(tA, TB[c], tB[c]);
    TA *= tA;
  }
}

// Backward pass with carry-in (from the rows above this segment), periodic correction -f_c z;
// x overwrites y (ld ldy) and is copied to x2 (ld ldx2); per-column ||x||^2 partials into nrm.
__device__ inline void seg_bwd_multi(int g0, int cnt, const double* di, const double* cs, const double* fz,
                                     const double (&f)[CB], double* y, int ldy, double* x2, int ldx2, int nc,
                                     const double (&carry0)[CB], double* wsmM, double (&nrm)[CB]) {
  const int t = threadIdx.x;
  double carry[CB];
#pragma unroll
  for (int c = 0; c < CB; ++c) { carry[c] = carry0[c]; nrm[c] = 0.0; }
  for (int base = ((cnt - 1) / CHUNK) * CHUNK; base >= 0 && cnt > 0; base -= CHUNK) {
    double av[EPT], dvv[EPT], A = 1.0, B[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) B[c] = 0.0;
#pragma unroll
    for (int k = EPT - 1; k >= 0; --k) {
      const int i = base + t * EPT + k;
      dvv[k] = i < cnt ? di[g0 + i] : 0.0;
      av[k] = i < cnt ? -dvv[k] * cs[g0 + i] : 1.0;
      if (i < cnt) {
#pragma unroll
        for (int c = 0; c < CB; ++c) B[c] = fma(av[k], B[c], c < nc ? dvv[k] * y[size_t(c) * ldy + i] : 0.0);
        A *= av[k];
      }
    }
    double pA, pB[CB], tA, tB[CB];
    block_scan_multi<true>(A, B, wsmM, pA, pB, tA, tB);
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      if (c < nc) {
        double v = fma(pA, carry[c], pB[c]);
#pragma unroll
        for (int k = EPT - 1; k >= 0; --k) {
          const int i = base + t * EPT + k;
          if (i < cnt) {
            v = fma(av[k], v, dvv[k] * y[size_t(c) * ldy + i]);
            const double w = fz ? fma(-f[c], fz[g0 + i], v) : v;
            y[size_t(c) * ldy + i] = w;
            x2[size_t(c) * ldx2 + i] = w;
            nrm[c] = fma(w, w, nrm[c]);
          }
        }
      }
      carry[c] = fma(tA, carry[c], tB[c]);
    }
  }
}

// m columns W_c = (I - gamma A)^{-1} Vb_c on the cluster-split rows; W0 gets a copy; s.n0[c] =
// ||W_c||^2 (cluster-reduced).  xch layout (per column c < MB): [0,2MB) forward maps, [2MB,3MB)
// periodic dots, [3MB,5MB) backward maps, [5MB,6MB) norm partials.
template <int MB>
__device__ inline void cl_sai_solve(cg::cluster_group& cl, int cs, int cr, int ld, int g0, int cnt, int periodic,
                                    const double* l, const double* di, const double* sup, const double* fz,
                                    const double* fw, const double* Vb, int m, double* W, int ldw, double* W0,
                                    SmemT& s, double* wsmM, double* red) {
  double* xf = s.xch;
  double* xd = s.xch + 2 * MB;
  double* xb = s.xch + 3 * MB;
  double* xn = s.xch + 5 * MB;
  // ---- forward segment maps (+ the periodic Sherman-Morrison dots w'^T b)
  for (int c0 = 0; c0 < m; c0 += CB) {
    const int nc = min(CB, m - c0);
    double TA = 1.0, TB[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) TB[c] = 0.0;
    if (cs > 1 && cr < cs - 1) seg_maps_fwd(g0, cnt, l, Vb + size_t(c0) * ld, ld, nc, wsmM, TA, TB);
    if (threadIdx.x == 0)
      for (int c = 0; c < nc; ++c) { xf[2 * (c0 + c)] = TA; xf[2 * (c0 + c) + 1] = TB[c]; }
  }
  if (periodic)
    for (int c = 0; c < m; ++c) {
      double dot = 0.0;
      for (int i = threadIdx.x; i < cnt; i += PEXP_THREADS) dot = fma(fw[g0 + i], Vb[size_t(c) * ld + i], dot);
      dot = block_sum(dot, red);
      if (threadIdx.x == 0) xd[c] = dot;
    }
  else if (threadIdx.x < m)
    xd[threadIdx.x] = 0.0;
  cl_sync(cl, cs);
  __shared__ double carry_s[MB], f_s[MB];
  for (int c = threadIdx.x; c < m; c += PEXP_THREADS) {
    double carry = 0.0, f = 0.0;
    for (int q = 0; q < cs; ++q) {
      const double* rx = cs > 1 ? cl.map_shared_rank(s.xch, q) : s.xch;
      if (q < cr) carry = fma(rx[2 * c], carry, rx[2 * c + 1]);
      f += rx[2 * MB + c];
    }
    carry_s[c] = carry;
    f_s[c] = f;
  }
  __syncthreads();
  for (int c0 = 0; c0 < m; c0 += CB) {
    const int nc = min(CB, m - c0);
    double cin[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) cin[c] = c < nc ? carry_s[c0 + c] : 0.0;
    seg_fwd_multi(g0, cnt, l, Vb + size_t(c0) * ld, ld, W + size_t(c0) * ldw, ldw, nc, cin, wsmM);
  }
  __syncthreads();
  // ---- backward segment maps
  for (int c0 = 0; c0 < m; c0 += CB) {
    const int nc = min(CB, m - c0);
    double TA = 1.0, TB[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) TB[c] = 0.0;
    if (cs > 1 && cr > 0) seg_maps_bwd(g0, cnt, di, sup, W + size_t(c0) * ldw, ldw, nc, wsmM, TA, TB);
    if (threadIdx.x == 0)
      for (int c = 0; c < nc; ++c) { xb[2 * (c0 + c)] = TA; xb[2 * (c0 + c) + 1] = TB[c]; }
  }
  cl_sync(cl, cs);
  for (int c = threadIdx.x; c < m; c += PEXP_THREADS) {
    double carry = 0.0;
    for (int q = cs - 1; q > cr; --q) {
      const double* rx = cl.map_shared_rank(s.xch, q);
      carry = fma(rx[3 * MB + 2 * c], carry, rx[3 * MB + 2 * c + 1]);
    }
    carry_s[c] = carry;
  }
  __syncthreads();
  for (int c0 = 0; c0 < m; c0 += CB) {
    const int nc = min(CB, m - c0);
    double cin[CB], fc[CB], nrm[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) { cin[c] = c < nc ? carry_s[c0 + c] : 0.0; fc[c] = c < nc ? f_s[c0 + c] : 0.0; }
    seg_bwd_multi(g0, cnt, di, sup, periodic ? fz : nullptr, fc, W + size_t(c0) * ldw, ldw, W0 + size_t(c0) * ld,
                  ld, nc, cin, wsmM, nrm);
    // the nc column norms in one block reduction (warp shuffles, then warp partials in wsmM)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < CB; ++c) nrm[c] = warp_sum(nrm[c]);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < CB; ++c) wsmM[w * CB + c] = nrm[c];
    __syncthreads();
    if (threadIdx.x < nc) {
      double v = 0.0;
      for (int k = 0; k < PEXP_THREADS / 32; ++k) v += wsmM[k * CB + threadIdx.x];
      xn[c0 + threadIdx.x] = v;
    }
    __syncthreads();
  }
  cl_allreduce(cl, cs, xn, s.n0, m);
}

template <int MB>
__global__ void __launch_bounds__(PEXP_THREADS, MB <= 8 ? 2 : 1) k_arnoldi_step(StepArgs A) {
  extern __shared__ double sm[];
  __shared__ double wsmM[(2 * (PEXP_THREADS / 32) + 1) * (CB + 1)];
  __shared__ double red[32];
  __shared__ int cls[MB], perm[MB], used[MB], dead[MB];
  cg::cluster_group cl = cg::this_cluster();
  const int cs = A.cs, cr = cs > 1 ? int(cl.block_rank()) : 0;
  const int e = blockIdx.x / cs;
  if (A.active && !A.active[e]) return;  // uniform over the cluster
  const int n = A.n, m = A.m, b = A.b, kcap = A.kcap, nv = (b + 1) * m;
  // this CTA's rows [g0, g0 + cnt) of every column (multiples of 32)
  const int per = step_rows(n, cs);
  const int g0 = min(n, cr * per), cnt = min(n, g0 + per) - g0;
  SmemT s;
  s.ldc = RC + 1;
  s.gpar = 0;
  const int cbuf = max(s.ldc * MB, PEXP_THREADS * SPAD);
  double* p = sm;
  const long long hst = (long long)nv * MB;   // V^T W partial / sum size
  double* Pp0 = nullptr;                      // rank-0 partial (global variant)
  if (A.hs_glob) {                            // [e][rank][2][nv*MB] in global memory
    s.Hs = A.hs_g + (size_t(e) * cs + cr) * 2 * hst;
    s.Pp = s.Hs + hst;
    Pp0 = A.hs_g + size_t(e) * cs * 2 * hst + hst;
  } else {
    s.Hs = p; p += hst;
    s.Pp = p; p += hst;
  }
  s.Cx = p; p += cbuf;
  s.Cy = p; p += cbuf;
  s.G = p; p += MB * MB;
  s.Gp = p; p += 2 * MB * MB;
  s.Rinv = p; p += MB * MB;
  s.Mc = p; p += MB * MB;
  s.S = p; p += MB * (MB + 1);
  s.Xw = p; p += MB * (MB + 1);
  s.Lp = p; p += MB * (MB + 1);
  s.d = p; p += MB;
  s.n0 = p; p += MB;
  s.n0p = p; p += MB;
  s.xch = p; p += 6 * MB;
  s.Ws = A.ws_smem ? p : nullptr;
  double* V = A.V + e * A.vs_e + g0;
  double* H = A.H + e * A.hs_e;
  int* live = A.live + size_t(e) * kcap;
  double* W0 = A.W0 + e * A.w0s_e + g0;
  double* Wg = V + size_t(nv) * n;              // the new block in the basis (global)
  double* W = A.ws_smem ? s.Ws : Wg;            // working copy of the CTA's rows
  const int ldw = A.ws_smem ? per : n;
  const size_t fo = size_t(A.fidx ? A.fidx[e] : e) * n;
  // ---- W0 = (I - gamma A)^{-1} V_b   (kept in W0; working copy in W)
  cl_sai_solve<MB>(cl, cs, cr, n, g0, cnt, A.periodic, A.fl + fo, A.fdinv + fo, A.fsup + fo,
                   A.periodic ? A.fz + fo : nullptr, A.periodic ? A.fw + fo : nullptr, V + size_t(b * m) * n, m, W,
                   ldw, W0, s, wsmM, red);
  // ---- BCGS pass 1
  cta_vtw<MB>(n, ldw, cnt, V, nv, W, m, s.Pp, s.Cx, s.ldc);
  if (A.hs_glob)
    cl_allreduce_g(cl, cs, Pp0, 2 * hst, s.Hs, nv * m);
  else
    cl_allreduce(cl, cs, s.Pp, s.Hs, nv * m);
  if (cr == 0)
    for (int i = threadIdx.x; i < nv * m; i += PEXP_THREADS) {
      int a = i % nv, c = i / nv;
      H[a + size_t(b * m + c) * kcap] = s.Hs[i];
    }
  cta_update<MB>(n, ldw, cnt, V, nv, W, m, s.Hs);
  // ---- in-block QR, stage A (accept kappa <= 1e4, defer the rest, drop below defl*|W0|)
  cl_gram<MB>(cl, cs, ldw, ldw, cnt, W, W, m, s);
  const double pminA = cta_chol_piv<MB>(m, s.G, s.n0, A.defl, 1e-8, A.piv_tol, s, cls, perm, used, dead);
  cta_apply<MB>(ldw, cnt, W, m, s.Rinv, 0.0);
  // ---- stage B: explicit CGS2 of deferred columns against accepted ones (skipped when the
  // stage-A factorisation deferred nothing; cls is identical in every CTA of the cluster)
  __shared__ int s_ndef;
  if (threadIdx.x == 0) {
    int nd = 0;
    for (int k = 0; k < m; ++k) nd += cls[k] == 2;
    s_ndef = nd;
  }
  __syncthreads();
  for (int rep = 0; rep < (s_ndef > 0 ? 2 : 0); ++rep) {
    cl_gram<MB>(cl, cs, ldw, ldw, cnt, W, W, m, s);
    for (int idx = threadIdx.x; idx < MB * MB; idx += PEXP_THREADS) {
      int a = idx % MB, k = idx / MB;
      s.Mc[idx] = (a < m && k < m && cls[a] == 1 && cls[k] == 2) ? -s.G[a + k * MB] : 0.0;
    }
    __syncthreads();
    cta_apply<MB>(ldw, cnt, W, m, s.Mc, 1.0);
  }
  // ---- stage C: final pivoted CholQR with deflation relative to |W0|.  Skipped when stage A
  // accepted every column with scaled pivots >= 1e-2 (scaled Gram condition <= ~1e2, so one
  // CholQR left the block orthonormal to ~1e-12 and BCGS pass 2 + its CholQR finish the job);
  // the decision uses cluster-identical data.
  __shared__ int s_nacc;
  if (threadIdx.x == 0) {
    int na = 0;
    for (int k = 0; k < m; ++k) na += cls[k] == 1;
    s_nacc = na;
  }
  __syncthreads();
  if (!(s_ndef == 0 && s_nacc == m && pminA >= 1e-2)) {
    cl_gram<MB>(cl, cs, ldw, ldw, cnt, W, W, m, s);
    for (int k = threadIdx.x; k < m; k += PEXP_THREADS) s.n0[k] = s.n0p[k];
    __syncthreads();
    cta_chol_piv<MB>(m, s.G, s.n0, A.defl, 0.0, A.piv_tol, s, cls, perm, used, dead);
    cta_apply<MB>(ldw, cnt, W, m, s.Rinv, 0.0);
  }
  // ---- BCGS pass 2 + CholQR
  cta_vtw<MB>(n, ldw, cnt, V, nv, W, m, s.Pp, s.Cx, s.ldc);
  if (A.hs_glob)
    cl_allreduce_g(cl, cs, Pp0, 2 * hst, s.Hs, nv * m);
  else
    cl_allreduce(cl, cs, s.Pp, s.Hs, nv * m);
  cta_update<MB>(n, ldw, cnt, V, nv, W, m, s.Hs);
  cl_gram<MB>(cl, cs, ldw, ldw, cnt, W, W, m, s);
  cta_chol_piv<MB>(m, s.G, nullptr, A.defl, 0.0, A.piv_tol, s, cls, perm, used, dead);
  cta_apply<MB>(ldw, cnt, W, m, s.Rinv, 0.0);
  // ---- the new basis block to global memory; subdiagonal block H[nv + a, b*m + c] = Q_a^T W0_c
  if (A.ws_smem)
    for (int idx = threadIdx.x; idx < m * cnt; idx += PEXP_THREADS) {
      const int c = idx / cnt, r = idx % cnt;
      Wg[size_t(c) * n + r] = W[size_t(c) * ldw + r];
    }
  cl_gram<MB>(cl, cs, ldw, n, cnt, W, W0, m, s);
  if (cr == 0) {
    for (int i = threadIdx.x; i < m * m; i += PEXP_THREADS) {
      int a = i % m, c = i / m;
      H[nv + a + size_t(b * m + c) * kcap] = s.G[a + c * MB];
    }
    for (int k = threadIdx.x; k < m; k += PEXP_THREADS) live[nv + k] = cls[k] ? 1 : 0;
  }
  cl_sync(cl, cs);  // no CTA leaves while its shared memory may still be read remotely
}

static size_t step_smem(int MB, int nv, int wrows) {
  const int ldc = RC + 1;
  size_t cbuf = std::max(size_t(ldc) * MB, size_t(PEXP_THREADS) * SPAD);
  return sizeof(double) * (2 * size_t(nv) * MB + 2 * cbuf + 5 * MB * MB + 3 * MB * (MB + 1) + 3 * MB + 6 * MB +
                           size_t(wrows) * MB);
}

static int mb_for(int m) { return m <= 8 ? 8 : (m <= 16 ? 16 : 32); }

static int step_cluster(int E, int n);

// The fused step is used when the CTA's rows of the new block fit shared memory (the V^T W
// partials may live in global scratch).  Otherwise (very long columns, e.g. C5's 8192 rows per
// CTA) the multi-kernel route streams V with full-grid launches, which measured 2x faster there.
bool arnoldi_fused_ok(int m, int nv, int n, int E, bool have_global_scratch) {
  if (m > 32) return false;
  const int MB = mb_for(m), per = step_rows(n, step_cluster(E, n));
  if (step_smem(MB, nv, per) <= 200 * 1024) return true;
  return have_global_scratch && step_smem(MB, 0, per) <= 200 * 1024;
}

// global scratch of the fused step for E evaluations (clusters of <= 8 CTAs, nv <= kcap)
size_t arnoldi_scratch_doubles(int E, int kcap, int mcap) {
  const int MB = mb_for(std::min(mcap, 32));
  if (step_smem(MB, kcap, 0) <= 200 * 1024) return 0;  // every step fits shared memory
  return size_t(E) * 16 * 2 * size_t(kcap) * MB;
}

// cluster size: enough CTAs for ~2 waves over the 148 SMs, >= 512 rows per CTA, portable max 8
static int step_cluster(int E, int n) {
  int cs = 1;
  while (cs < 8 && long(E) * cs < 2 * 148 && n / (2 * cs) >= 512) cs *= 2;
  // very small batches (e.g. 8 groups of homogeneous legs): a non-portable 16-CTA cluster
  if (cs == 8 && E * 16 <= 148 && n / 16 >= 256) cs = 16;
  return cs;
}

template <int MB>
static void launch_mb(cudaStream_t st, const StepArgs& a, size_t smem) {
  cudaFuncSetAttribute(k_arnoldi_step<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (a.cs > 1) cudaFuncSetAttribute(k_arnoldi_step<MB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.E * a.cs);
  cfg.blockDim = dim3(PEXP_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PEXP_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_arnoldi_step<MB>, a));
}

void launch_arnoldi_step(cudaStream_t st, StepArgs a) {
  const int MB = mb_for(a.m);
  a.rc = RC;
  a.piv_tol = g_cfg.piv_tol;
  a.cs = step_cluster(a.E, a.n);
  const int nv = (a.b + 1) * a.m;
  const int per = step_rows(a.n, a.cs);
  size_t smem = step_smem(MB, nv, per);
  a.ws_smem = 1;  // the CTA's rows of the new block stay on chip
  a.hs_glob = 0;
  if (smem > 200 * 1024) {  // V^T W partials and sums to global memory (large Krylov dimensions)
    if (!a.hs_g) fail(1, "fused Arnoldi step: no global scratch for a large basis");
    a.hs_glob = 1;
    smem = step_smem(MB, 0, per);
  }
  if (smem > 200 * 1024) fail(1, "fused Arnoldi step: block rows exceed shared memory");
  const double ea = eact(a.E, a.active);
  ProfScope ps(PC_ARNOLDI, st, ea * a.n * 8.0 * (4.0 * nv + 12.0 * a.m), ea * a.n * (8.0 * nv * a.m + 10.0 * a.m * a.m));
  if (MB == 8)
    launch_mb<8>(st, a, smem);
  else if (MB == 16)
    launch_mb<16>(st, a, smem);
  else
    launch_mb<32>(st, a, smem);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

}  // namespace pexp
