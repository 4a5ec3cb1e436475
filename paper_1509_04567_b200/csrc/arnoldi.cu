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

// ---------------------------------------------------------------- cluster-split SaI solve
// Forward L-solve y_g = -l_g y_{g-1} + b_g and backward U-solve x_g = -d_g c_g x_{g+1} + d_g y_g
// as affine maps (scan.cuh).  Rows [g0, g0 + cnt) belong to this CTA; each thread composes EPT
// consecutive rows of a CHUNK, a block scan composes the threads.
__device__ inline Aff seg_map_fwd(int g0, int cnt, const double* l, const double* b, Aff* wsm) {
  const int t = threadIdx.x;
  Aff acc{1.0, 0.0};
  for (int base = 0; base < cnt; base += CHUNK) {
    Aff mp{1.0, 0.0};
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = base + t * EPT + k;
      if (i < cnt) mp = after(mp, Aff{-l[g0 + i], b[i]});
    }
    Aff tot;
    block_excl_scan<false>(mp, t, wsm, tot);
    acc = after(acc, tot);
  }
  return acc;
}

__device__ inline Aff seg_map_bwd(int g0, int cnt, const double* di, const double* cs, const double* y, Aff* wsm) {
  const int t = threadIdx.x;
  Aff acc{1.0, 0.0};
  for (int base = ((cnt - 1) / CHUNK) * CHUNK; base >= 0 && cnt > 0; base -= CHUNK) {
    Aff mp{1.0, 0.0};
#pragma unroll
    for (int k = EPT - 1; k >= 0; --k) {
      const int i = base + t * EPT + k;
      if (i < cnt) {
        const double dv = di[g0 + i];
        mp = after(mp, Aff{-dv * cs[g0 + i], dv * y[i]});
      }
    }
    Aff tot;
    block_excl_scan<true>(mp, PEXP_THREADS - 1 - t, wsm, tot);
    acc = after(acc, tot);
  }
  return acc;
}

// Forward pass with carry-in: y[i] (own rows) from b[i]; returns nothing (y written to out).
__device__ inline void seg_fwd(int g0, int cnt, const double* l, const double* b, double* y, double carry, double* s0,
                               double* s1, Aff* wsm) {
  const int t = threadIdx.x;
  for (int base = 0; base < cnt; base += CHUNK) {
    for (int i = t; i < CHUNK; i += PEXP_THREADS) {
      const int g = base + i;
      const int si = (i / EPT) * SPAD + (i % EPT);
      s0[si] = g < cnt ? b[g] : 0.0;
      s1[si] = g < cnt ? -l[g0 + g] : 1.0;
    }
    __syncthreads();
    Aff mp{1.0, 0.0};
#pragma unroll
    for (int k = 0; k < EPT; ++k) mp = after(mp, Aff{s1[t * SPAD + k], s0[t * SPAD + k]});
    Aff tot;
    Aff pre = block_excl_scan<false>(mp, t, wsm, tot);
    double v = fma(pre.A, carry, pre.B);
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      v = fma(s1[t * SPAD + k], v, s0[t * SPAD + k]);
      s0[t * SPAD + k] = v;
    }
    carry = fma(tot.A, carry, tot.B);
    __syncthreads();
    for (int i = t; i < CHUNK; i += PEXP_THREADS) {
      const int g = base + i;
      if (g < cnt) y[g] = s0[(i / EPT) * SPAD + (i % EPT)];
    }
    __syncthreads();
  }
}

// Backward pass with carry-in (from the rows above this segment), periodic correction -f*z;
// writes x into x and x2; returns this CTA's partial ||x||^2 (block-reduced).
__device__ inline double seg_bwd(int g0, int cnt, const double* di, const double* cs, const double* fz, double f,
                                 double* x, double* x2, double carry, double* s0, double* s1, Aff* wsm, double* red) {
  const int t = threadIdx.x;
  double nrm2 = 0.0;
  for (int base = ((cnt - 1) / CHUNK) * CHUNK; base >= 0 && cnt > 0; base -= CHUNK) {
    for (int i = t; i < CHUNK; i += PEXP_THREADS) {
      const int g = base + i;
      const int si = (i / EPT) * SPAD + (i % EPT);
      if (g < cnt) {
        const double dv = di[g0 + g];
        s0[si] = dv * x[g];
        s1[si] = -dv * cs[g0 + g];
      } else {
        s0[si] = 0.0;
        s1[si] = 1.0;
      }
    }
    __syncthreads();
    Aff mp{1.0, 0.0};
#pragma unroll
    for (int k = EPT - 1; k >= 0; --k) mp = after(mp, Aff{s1[t * SPAD + k], s0[t * SPAD + k]});
    Aff tot;
    Aff pre = block_excl_scan<true>(mp, PEXP_THREADS - 1 - t, wsm, tot);
    double v = fma(pre.A, carry, pre.B);
#pragma unroll
    for (int k = EPT - 1; k >= 0; --k) {
      v = fma(s1[t * SPAD + k], v, s0[t * SPAD + k]);
      s0[t * SPAD + k] = v;
    }
    carry = fma(tot.A, carry, tot.B);
    __syncthreads();
    for (int i = t; i < CHUNK; i += PEXP_THREADS) {
      const int g = base + i;
      if (g < cnt) {
        double w = s0[(i / EPT) * SPAD + (i % EPT)];
        if (fz) w = fma(-f, fz[g0 + g], w);
        x[g] = w;
        x2[g] = w;
        nrm2 = fma(w, w, nrm2);
      }
    }
    __syncthreads();
  }
  return block_sum(nrm2, red);
}

// m columns W_c = (I - gamma A)^{-1} Vb_c on the cluster-split rows; W0 gets a copy; s.n0[c] =
// ||W_c||^2 (cluster-reduced).  xch layout: [0,2MB) forward maps, [2MB,3MB) periodic dots,
// [3MB,5MB) backward maps, [5MB,6MB) norm partials; s.Gp scratch for the reduced norms.
template <int MB>
__device__ inline void cl_sai_solve(cg::cluster_group& cl, int cs, int cr, int ld, int g0, int cnt, int periodic,
                                    const double* l, const double* di, const double* sup, const double* fz,
                                    const double* fw, const double* Vb, int m, double* W, int ldw, double* W0,
                                    SmemT& s, Aff* wsm, double* red) {
  double* xf = s.xch;
  double* xd = s.xch + 2 * MB;
  double* xb = s.xch + 3 * MB;
  double* xn = s.xch + 5 * MB;
  // ---- forward segment maps (+ the periodic Sherman-Morrison dots w'^T b)
  for (int c = 0; c < m; ++c) {
    const double* b = Vb + size_t(c) * ld;
    Aff F = (cs > 1 && cr < cs - 1) ? seg_map_fwd(g0, cnt, l, b, wsm) : Aff{1.0, 0.0};
    double dot = 0.0;
    if (periodic)
      for (int i = threadIdx.x; i < cnt; i += PEXP_THREADS) dot = fma(fw[g0 + i], b[i], dot);
    dot = periodic ? block_sum(dot, red) : 0.0;
    if (threadIdx.x == 0) { xf[2 * c] = F.A; xf[2 * c + 1] = F.B; xd[c] = dot; }
  }
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
  for (int c = 0; c < m; ++c) seg_fwd(g0, cnt, l, Vb + size_t(c) * ld, W + size_t(c) * ldw, carry_s[c], s.Cx, s.Cy, wsm);
  // ---- backward segment maps
  for (int c = 0; c < m; ++c) {
    Aff Bm = (cs > 1 && cr > 0) ? seg_map_bwd(g0, cnt, di, sup, W + size_t(c) * ldw, wsm) : Aff{1.0, 0.0};
    if (threadIdx.x == 0) { xb[2 * c] = Bm.A; xb[2 * c + 1] = Bm.B; }
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
  for (int c = 0; c < m; ++c) {
    double nr = seg_bwd(g0, cnt, di, sup, periodic ? fz : nullptr, f_s[c], W + size_t(c) * ldw, W0 + size_t(c) * ld,
                        carry_s[c], s.Cx, s.Cy, wsm, red);
    if (threadIdx.x == 0) xn[c] = nr;
  }
  cl_allreduce(cl, cs, xn, s.n0, m);
}

template <int MB>
__global__ void __launch_bounds__(PEXP_THREADS) k_arnoldi_step(StepArgs A) {
  extern __shared__ double sm[];
  __shared__ Aff wsm[PEXP_THREADS / 32 + 1];
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
  s.Hs = p; p += size_t(nv) * MB;
  s.Pp = p; p += size_t(nv) * MB;
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
                   ldw, W0, s, wsm, red);
  // ---- BCGS pass 1
  cta_vtw<MB>(n, ldw, cnt, V, nv, W, m, s.Pp, s.Cx, s.ldc);
  cl_allreduce(cl, cs, s.Pp, s.Hs, nv * m);
  if (cr == 0)
    for (int i = threadIdx.x; i < nv * m; i += PEXP_THREADS) {
      int a = i % nv, c = i / nv;
      H[a + size_t(b * m + c) * kcap] = s.Hs[i];
    }
  cta_update<MB>(n, ldw, cnt, V, nv, W, m, s.Hs);
  // ---- in-block QR, stage A (accept kappa <= 1e4, defer the rest, drop below defl*|W0|)
  cl_gram<MB>(cl, cs, ldw, ldw, cnt, W, W, m, s);
  cta_chol_piv<MB>(m, s.G, s.n0, A.defl, 1e-8, A.piv_tol, s, cls, perm, used, dead);
  cta_apply<MB>(ldw, cnt, W, m, s.Rinv, 0.0);
  // ---- stage B: explicit CGS2 of deferred columns against accepted ones
  for (int rep = 0; rep < 2; ++rep) {
    cl_gram<MB>(cl, cs, ldw, ldw, cnt, W, W, m, s);
    for (int idx = threadIdx.x; idx < MB * MB; idx += PEXP_THREADS) {
      int a = idx % MB, k = idx / MB;
      s.Mc[idx] = (a < m && k < m && cls[a] == 1 && cls[k] == 2) ? -s.G[a + k * MB] : 0.0;
    }
    __syncthreads();
    cta_apply<MB>(ldw, cnt, W, m, s.Mc, 1.0);
  }
  // ---- stage C: final pivoted CholQR with deflation relative to |W0|
  cl_gram<MB>(cl, cs, ldw, ldw, cnt, W, W, m, s);
  for (int k = threadIdx.x; k < m; k += PEXP_THREADS) s.n0[k] = s.n0p[k];
  __syncthreads();
  cta_chol_piv<MB>(m, s.G, s.n0, A.defl, 0.0, A.piv_tol, s, cls, perm, used, dead);
  cta_apply<MB>(ldw, cnt, W, m, s.Rinv, 0.0);
  // ---- BCGS pass 2 + CholQR
  cta_vtw<MB>(n, ldw, cnt, V, nv, W, m, s.Pp, s.Cx, s.ldc);
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

bool arnoldi_fused_ok(int m, int nv) {
  if (m > 32) return false;
  return step_smem(mb_for(m), nv, 0) <= 200 * 1024;
}

// cluster size: enough CTAs for ~2 waves over the 148 SMs, >= 512 rows per CTA, portable max 8
static int step_cluster(int E, int n) {
  static const int force = getenv("PEXP_ACL") ? atoi(getenv("PEXP_ACL")) : 0;  // developer override
  if (force > 0) return force;
  int cs = 1;
  while (cs < 8 && long(E) * cs < 2 * 148 && n / (2 * cs) >= 512) cs *= 2;
  return cs;
}

extern double g_piv_tol;

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
  a.piv_tol = g_piv_tol;
  a.cs = step_cluster(a.E, a.n);
  const int nv = (a.b + 1) * a.m;
  const int per = step_rows(a.n, a.cs);
  size_t smem = step_smem(MB, nv, per);
  a.ws_smem = smem <= 200 * 1024 ? 1 : 0;  // the CTA's rows of the new block stay on chip
  if (!a.ws_smem) smem = step_smem(MB, nv, 0);
  ProfScope ps(PC_ARNOLDI, st, double(a.E) * a.n * 8.0 * (4.0 * nv + 12.0 * a.m),
               double(a.E) * a.n * (8.0 * nv * a.m + 10.0 * a.m * a.m));
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
