// dense.cuh — CTA-level dense fp64 linear algebra on small matrices (N <= ~600) held in
// global memory (L2-resident per-evaluation workspace).  Every routine is called by ALL
// threads of the CTA and contains the needed __syncthreads().  Column-major storage.
#pragma once
#include "common.cuh"

namespace pexp {

// A group of CTAs cooperating on one evaluation: a thread-block cluster (rank, size), or a
// single CTA (size 1).  Operands live in global memory (L2), so a cluster barrier with
// release/acquire semantics (plus a device-scope fence) orders the phases.
struct Grp {
  int rank, size;
};

__device__ inline Grp this_grp() {
  unsigned r, s;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(s));
  return Grp{int(r), int(s)};
}

__device__ inline void grp_sync(const Grp& g) {
  if (g.size == 1) {
    __syncthreads();
    return;
  }
  __threadfence();
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr Grp kSolo{0, 1};

// C = alpha*A*B + beta*C ; A: M x K (lda), B: K x N (ldb), C: M x N (ldc); C must not alias.
// Tiles TM x TM (TM = 128 or 64) with K-steps of 16 staged in shared memory; 256 threads as a
// 16 x 16 grid, each owning (TM/16)^2 outputs strided by 16 (conflict-free shared reads, 4 FMA
// per shared load at TM = 128; the thread's row index runs fastest across a warp so the epilogue's
// C reads/writes are coalesced); the next K-step is prefetched into registers while the current
// one is consumed (hides the L2 latency of these L2-resident operands).
// one shared staging buffer per kernel, shared by both tile instantiations
// PEXP_GEMM_TM: largest CTA tile of the dense routines (64 keeps the projected-problem kernels at
// <= 128 registers and ~95 KB of shared memory, i.e. two CTAs per SM)
#ifndef PEXP_GEMM_TM
#define PEXP_GEMM_TM 64
#endif
__device__ inline double* gemm_smem() {
  __shared__ __align__(16) double buf[2 * 16 * (PEXP_GEMM_TM + 8)];
  return buf;
}

// fp64 tensor-core MMA (DMMA): D(8x8) += A(8x4, row) B(4x8, col); per lane: A[lane/4][lane%4],
// B[lane%4][lane/4], D[lane/4][2(lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Same contract as cta_gemm_t, on the fp64 tensor cores: TM x TM CTA tiles, 8 warps as 4 (rows) x 2
// (columns), warp tile (TM/4) x (TM/2) of m8n8 accumulators, K-steps of 16 staged in shared memory
// (rows padded to TM + 8 doubles: the 4 k-rows of a fragment load fall in disjoint banks), the next
// K-step prefetched into registers.
template <int TM>
__device__ inline void cta_gemm_dmma(int M, int N, int K, double alpha, const double* A, int lda, const double* B,
                                     int ldb, double beta, double* C, int ldc, Grp g) {
  constexpr int LDS = TM + 8;
  constexpr int WM = TM / 4, WN = TM / 2, MI = WM / 8, NI = WN / 8;
  constexpr int LA = TM * 16 / 256;
  double (*As)[LDS] = reinterpret_cast<double (*)[LDS]>(gemm_smem());
  double (*Bs)[LDS] = reinterpret_cast<double (*)[LDS]>(gemm_smem() + 16 * LDS);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, wm = warp & 3, wn = warp >> 2;
  const int fr = lane >> 2, fc = lane & 3;
  const int nti = (M + TM - 1) / TM, ntj = (N + TM - 1) / TM;
  for (int tile = g.rank; tile < nti * ntj; tile += g.size) {
    const int i0 = (tile % nti) * TM, j0 = (tile / nti) * TM;
    double acc[MI][NI][2];
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int b = 0; b < NI; ++b) { acc[a][b][0] = 0.0; acc[a][b][1] = 0.0; }
    double pa[LA], pb[LA];
    auto load = [&](int k0) {
#pragma unroll
      for (int q = 0; q < LA; ++q) {
        int idx = t + q * 256;
        int r = idx % TM, kk = idx / TM;        // A: rows fastest (coalesced)
        int gi = i0 + r, gk = k0 + kk;
        pa[q] = (gi < M && gk < K) ? A[gi + size_t(gk) * lda] : 0.0;
        int kb = idx % 16, c = idx / 16;        // B: k fastest within a column
        int gkb = k0 + kb, gj = j0 + c;
        pb[q] = (gkb < K && gj < N) ? B[gkb + size_t(gj) * ldb] : 0.0;
      }
    };
    load(0);
    for (int k0 = 0; k0 < K; k0 += 16) {
      __syncthreads();
#pragma unroll
      for (int q = 0; q < LA; ++q) {
        int idx = t + q * 256;
        As[idx / TM][idx % TM] = pa[q];
        Bs[idx % 16][idx / 16] = pb[q];
      }
      __syncthreads();
      if (k0 + 16 < K) load(k0 + 16);
#pragma unroll
      for (int kq = 0; kq < 4; ++kq) {
        double af[MI], bf[NI];
#pragma unroll
        for (int a = 0; a < MI; ++a) af[a] = As[kq * 4 + fc][wm * WM + a * 8 + fr];
#pragma unroll
        for (int b = 0; b < NI; ++b) bf[b] = Bs[kq * 4 + fc][wn * WN + b * 8 + fr];
#pragma unroll
        for (int a = 0; a < MI; ++a)
#pragma unroll
          for (int b = 0; b < NI; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
    }
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
      for (int b = 0; b < NI; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gi = i0 + wm * WM + a * 8 + fr, gj = j0 + wn * WN + b * 8 + 2 * fc + h;
          if (gi < M && gj < N) {
            double* c = C + gi + size_t(gj) * ldc;
            double v = alpha * acc[a][b][h];
            if (beta != 0.0) v = fma(beta, *c, v);
            *c = v;
          }
        }
  }
  grp_sync(g);
}

template <int TM>
__device__ inline void cta_gemm_t(int M, int N, int K, double alpha, const double* A, int lda, const double* B,
                                  int ldb, double beta, double* C, int ldc, Grp g) {
  constexpr int R = TM / 16;          // outputs per thread per dimension
  constexpr int LA = TM * 16 / 256;   // A-tile elements loaded per thread
  double (*As)[TM + 1] = reinterpret_cast<double (*)[TM + 1]>(gemm_smem());
  double (*Bs)[TM + 1] = reinterpret_cast<double (*)[TM + 1]>(gemm_smem() + 16 * (TM + 1));
  const int t = threadIdx.x, tx = t % 16, ty = t / 16;
  const int nti = (M + TM - 1) / TM, ntj = (N + TM - 1) / TM;
  for (int tile = g.rank; tile < nti * ntj; tile += g.size) {
    const int i0 = (tile % nti) * TM, j0 = (tile / nti) * TM;
    {
      double acc[R][R];
#pragma unroll
      for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < R; ++b) acc[a][b] = 0.0;
      double pa[LA], pb[LA];
      auto load = [&](int k0) {
#pragma unroll
        for (int q = 0; q < LA; ++q) {
          int idx = t + q * 256;
          int r = idx % TM, kk = idx / TM;        // A: rows fastest (coalesced)
          int gi = i0 + r, gk = k0 + kk;
          pa[q] = (gi < M && gk < K) ? A[gi + size_t(gk) * lda] : 0.0;
          int kb = idx % 16, c = idx / 16;        // B: k fastest within a column
          int gkb = k0 + kb, gj = j0 + c;
          pb[q] = (gkb < K && gj < N) ? B[gkb + size_t(gj) * ldb] : 0.0;
        }
      };
      load(0);
      for (int k0 = 0; k0 < K; k0 += 16) {
        __syncthreads();
#pragma unroll
        for (int q = 0; q < LA; ++q) {
          int idx = t + q * 256;
          As[idx / TM][idx % TM] = pa[q];
          Bs[idx % 16][idx / 16] = pb[q];
        }
        __syncthreads();
        if (k0 + 16 < K) load(k0 + 16);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          double av[R], bv[R];
#pragma unroll
          for (int a = 0; a < R; ++a) av[a] = As[kk][tx + 16 * a];
#pragma unroll
          for (int b = 0; b < R; ++b) bv[b] = Bs[kk][ty + 16 * b];
#pragma unroll
          for (int a = 0; a < R; ++a)
#pragma unroll
            for (int b = 0; b < R; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
      }
#pragma unroll
      for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < R; ++b) {
          int gi = i0 + tx + 16 * a, gj = j0 + ty + 16 * b;  // consecutive threads: consecutive rows
          if (gi < M && gj < N) {
            double* c = C + gi + size_t(gj) * ldc;
            double v = alpha * acc[a][b];
            if (beta != 0.0) v = fma(beta, *c, v);
            *c = v;
          }
        }
    }
  }
  grp_sync(g);
}

// 1: the fp64 tensor-core path (default); 0: SIMT FMA tiles (per translation unit; small.cu sets
// its copy from the developer switch PEXP_NODMMA)
static __device__ int g_gemm_dmma = 1;

__device__ inline void cta_gemm(int M, int N, int K, double alpha, const double* A, int lda, const double* B,
                                int ldb, double beta, double* C, int ldc, Grp g = kSolo) {
  // 128 x 128 tiles unless that leaves CTAs of the group without a tile
  const bool big = PEXP_GEMM_TM >= 128 && M > 64 && N > 64 && ((M + 127) / 128) * ((N + 127) / 128) >= g.size;
  if (g_gemm_dmma) {
    if (big)
      cta_gemm_dmma<PEXP_GEMM_TM>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, g);
    else
      cta_gemm_dmma<64>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, g);
    return;
  }
  if (big)
    cta_gemm_t<PEXP_GEMM_TM>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, g);
  else
    cta_gemm_t<64>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, g);
}

// Y = alpha*X + beta*Y (+ gamma*I) on N x N
__device__ inline void cta_axpby(int N, double alpha, const double* X, int ldx, double beta,
                                 double* Y, int ldy, double diag_add = 0.0, Grp g = kSolo) {
  for (int idx = threadIdx.x + g.rank * blockDim.x; idx < N * N; idx += blockDim.x * g.size) {
    int i = idx % N, j = idx / N;
    double v = alpha * X[i + size_t(j) * ldx] + (beta != 0.0 ? beta * Y[i + size_t(j) * ldy] : 0.0);
    if (i == j) v += diag_add;
    Y[i + size_t(j) * ldy] = v;
  }
  grp_sync(g);
}

__device__ inline void cta_copy(int M, int N, const double* X, int ldx, double* Y, int ldy, Grp g = kSolo) {
  for (int idx = threadIdx.x + g.rank * blockDim.x; idx < M * N; idx += blockDim.x * g.size) {
    int i = idx % M, j = idx / M;
    Y[i + size_t(j) * ldy] = X[i + size_t(j) * ldx];
  }
  grp_sync(g);
}

__device__ inline void cta_identity(int N, double* Y, int ldy, double d = 1.0, Grp g = kSolo) {
  for (int idx = threadIdx.x + g.rank * blockDim.x; idx < N * N; idx += blockDim.x * g.size) {
    int i = idx % N, j = idx / N;
    Y[i + size_t(j) * ldy] = (i == j) ? d : 0.0;
  }
  grp_sync(g);
}

// max column abs-sum: one warp per column, lanes over rows (coalesced, 4 loads in flight per lane)
__device__ inline double cta_norm1(int N, const double* A, int lda, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double mx = 0.0;
  for (int j = w; j < N; j += nw) {
    const double* col = A + size_t(j) * lda;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = lane;
    for (; i + 96 < N; i += 128) {
      s0 += fabs(col[i]); s1 += fabs(col[i + 32]); s2 += fabs(col[i + 64]); s3 += fabs(col[i + 96]);
    }
    for (; i < N; i += 32) s0 += fabs(col[i]);
    mx = fmax(mx, warp_sum((s0 + s1) + (s2 + s3)));
  }
  return block_max(mx, red);
}

// Triangular solve with a kb x kb (kb <= 32) diagonal block T (ld ldt) staged in shared memory:
// X (kb x ncols, ld ldx) <- T^{-1} X, unit lower (LOWER) or non-unit upper (!LOWER).  One thread
// per column keeps its kb values in registers.  Columns [c0, c1) of X; all CTA threads call it.
template <bool LOWER>
__device__ inline void cta_trsm_small(int kb, const double* T, int ldt, double* X, int ldx, int c0, int c1) {
  double (*Ts)[33] = reinterpret_cast<double (*)[33]>(gemm_smem());
  __syncthreads();
  for (int idx = threadIdx.x; idx < kb * kb; idx += blockDim.x) {
    const int i = idx % kb, j = idx / kb;
    Ts[i][j] = T[i + size_t(j) * ldt];
  }
  __syncthreads();
  for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
    double x[32];
    double* col = X + size_t(j) * ldx;
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = i < kb ? col[i] : 0.0;
    if (LOWER) {
#pragma unroll
      for (int i = 1; i < 32; ++i) {
        double v = x[i];
#pragma unroll
        for (int p = 0; p < i; ++p) v = fma(-Ts[i][p], x[p], v);
        x[i] = v;
      }
    } else {
#pragma unroll
      for (int i = 31; i >= 0; --i) {
        if (i < kb) {
          double v = x[i];
#pragma unroll
          for (int p = i + 1; p < 32; ++p)
            if (p < kb) v = fma(-Ts[i][p], x[p], v);
          x[i] = v / Ts[i][i];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < kb) col[i] = x[i];
  }
  __syncthreads();
}

// Blocked right-looking LU with partial pivoting, in place.  piv[k] = row swapped with k.
// Returns false if a zero pivot was met.  The N x NBL panel is factored in shared memory (psm,
// psm_cap doubles; NBL = 32, halved until the panel fits) by rank 0 of the group; its row
// interchanges are then applied to the other columns by the whole group; U12 = L11^{-1} A12 by
// register triangular solves, A22 -= L21 U12 by the CTA-level GEMM.
__device__ inline bool cta_lu(int N, double* A, int lda, int* piv, double* red, Grp g, double* psm, int psm_cap) {
  __shared__ int s_ip;
  __shared__ int s_bad;
  __shared__ int s_idx[32];
  if (threadIdx.x == 0) s_bad = 0;
  int NBL = 32;
  while (NBL > 1 && size_t(N) * NBL > size_t(psm_cap)) NBL /= 2;
  for (int k0 = 0; k0 < N; k0 += NBL) {
    const int kb = min(NBL, N - k0), h = N - k0;
    if (g.rank == 0) {
      double* P = psm;  // panel rows k0..N-1, columns k0..k0+kb-1, column-major ld h
      for (int idx = threadIdx.x; idx < h * kb; idx += blockDim.x) {
        const int i = idx % h, c = idx / h;
        P[idx] = A[k0 + i + size_t(k0 + c) * lda];
      }
      __syncthreads();
      for (int k = 0; k < kb; ++k) {
        double best = -1.0;
        int bi = k;
        for (int i = k + threadIdx.x; i < h; i += blockDim.x) {
          const double v = fabs(P[i + size_t(k) * h]);
          if (v > best) { best = v; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          double ob = __shfl_xor_sync(0xffffffffu, best, o);
          int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if ((threadIdx.x & 31) == 0) { red[threadIdx.x >> 5] = best; s_idx[threadIdx.x >> 5] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
          const int nw = (blockDim.x + 31) >> 5;
          double b = red[0];
          int ii = s_idx[0];
          for (int w = 1; w < nw; ++w) {
            if (red[w] > b || (red[w] == b && s_idx[w] < ii)) { b = red[w]; ii = s_idx[w]; }
          }
          s_ip = ii;
          piv[k0 + k] = k0 + ii;
          if (!(b > 0.0)) s_bad = 1;
        }
        __syncthreads();
        const int ip = s_ip;
        if (ip != k)
          for (int c = threadIdx.x; c < kb; c += blockDim.x) {
            const double t = P[k + size_t(c) * h];
            P[k + size_t(c) * h] = P[ip + size_t(c) * h];
            P[ip + size_t(c) * h] = t;
          }
        __syncthreads();
        const double pv = P[k + size_t(k) * h];
        const double inv = pv != 0.0 ? 1.0 / pv : 0.0;
        for (int i = k + 1 + threadIdx.x; i < h; i += blockDim.x) P[i + size_t(k) * h] *= inv;
        __syncthreads();
        const int w = kb - (k + 1), hh = h - (k + 1);
        for (int idx = threadIdx.x; idx < w * hh; idx += blockDim.x) {
          const int i = k + 1 + idx % hh, c = k + 1 + idx / hh;
          P[i + size_t(c) * h] = fma(-P[i + size_t(k) * h], P[k + size_t(c) * h], P[i + size_t(c) * h]);
        }
        __syncthreads();
      }
      for (int idx = threadIdx.x; idx < h * kb; idx += blockDim.x) {
        const int i = idx % h, c = idx / h;
        A[k0 + i + size_t(k0 + c) * lda] = P[idx];
      }
    }
    grp_sync(g);
    // the panel's interchanges on all other columns (one thread per column, group-split; a gather
    // through shared memory with a serial composition of the swaps measured slower)
    for (int j = threadIdx.x + g.rank * blockDim.x; j < N; j += blockDim.x * g.size) {
      if (j >= k0 && j < k0 + kb) continue;
      double* col = A + size_t(j) * lda;
      for (int k = k0; k < k0 + kb; ++k) {
        const int ip = piv[k];
        if (ip != k) { const double t = col[k]; col[k] = col[ip]; col[ip] = t; }
      }
    }
    grp_sync(g);
    const int rest = N - (k0 + kb);
    if (rest > 0) {
      // U12 = L11^{-1} A12 (unit lower), columns split over the group
      const int per = (rest + g.size - 1) / g.size;
      const int c0 = k0 + kb + g.rank * per, c1 = min(N, c0 + per);
      cta_trsm_small<true>(kb, A + k0 + size_t(k0) * lda, lda, A + k0, lda, c0, c1);
      grp_sync(g);
      // A22 -= L21 U12
      cta_gemm(rest, rest, kb, -1.0, A + (k0 + kb) + size_t(k0) * lda, lda,
               A + k0 + size_t(k0 + kb) * lda, lda, 1.0, A + (k0 + kb) + size_t(k0 + kb) * lda, lda, g);
    }
  }
  grp_sync(g);
  return s_bad == 0;
}

// Solve (LU) X = P B in place on B (N x nrhs), blocked; uses cta_gemm for off-diagonal blocks.
__device__ inline void cta_lu_solve_local(int N, const double* LU, int lda, const int* piv, double* B,
                                          int ldb, int nrhs, double* psm, int psm_cap, bool identity_rhs,
                                          int cbase);

// RHS columns are split into contiguous ranges, one per CTA of the group.  identity_rhs: B is
// the identity on entry (H^{-1}): P B is then written directly instead of permuted.
__device__ inline void cta_lu_solve(int N, const double* LU, int lda, const int* piv, double* B, int ldb, int nrhs,
                                    Grp g, double* psm, int psm_cap, bool identity_rhs = false) {
  const int per = (nrhs + g.size - 1) / g.size;
  const int c0 = g.rank * per, c1 = min(nrhs, c0 + per);
  cta_lu_solve_local(N, LU, lda, piv, B + size_t(c0) * ldb, ldb, max(0, c1 - c0), psm, psm_cap, identity_rhs, c0);
  grp_sync(g);
}

__device__ inline void cta_lu_solve_local(int N, const double* LU, int lda, const int* piv, double* B,
                                          int ldb, int nrhs, double* psm, int psm_cap, bool identity_rhs,
                                          int cbase) {
  // row order of P B: perm = the interchanges applied to 0..N-1 (thread 0, shared memory)
  int* perm = reinterpret_cast<int*>(psm);
  const int pint = (N + 1) / 2 + 1;  // doubles occupied by perm
  if (threadIdx.x == 0) {
    for (int i = 0; i < N; ++i) perm[i] = i;
    for (int k = 0; k < N; ++k) {
      const int ip = piv[k];
      if (ip != k) { const int t = perm[k]; perm[k] = perm[ip]; perm[ip] = t; }
    }
  }
  __syncthreads();
  if (nrhs > 0) {
    if (identity_rhs) {
      // B holds columns cbase.. of I: (P I)[i][j] = (perm[i] == cbase + j)
      const int c0 = cbase;
      for (int idx = threadIdx.x; idx < N * nrhs; idx += blockDim.x) {
        const int i = idx % N, j = idx / N;
        B[i + size_t(j) * ldb] = perm[i] == c0 + j ? 1.0 : 0.0;
      }
    } else {
      double* buf = psm + pint;
      const int cb = max(1, (psm_cap - pint) / max(N, 1));
      for (int j0 = 0; j0 < nrhs; j0 += cb) {
        const int nc = min(cb, nrhs - j0);
        for (int idx = threadIdx.x; idx < N * nc; idx += blockDim.x) {
          const int i = idx % N, j = idx / N;
          buf[idx] = B[perm[i] + size_t(j0 + j) * ldb];
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < N * nc; idx += blockDim.x) {
          const int i = idx % N, j = idx / N;
          B[i + size_t(j0 + j) * ldb] = buf[idx];
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  constexpr int NBL = 32;
  // forward: unit lower
  for (int k0 = 0; k0 < N; k0 += NBL) {
    const int kb = min(NBL, N - k0);
    cta_trsm_small<true>(kb, LU + k0 + size_t(k0) * lda, lda, B + k0, ldb, 0, nrhs);
    const int rest = N - (k0 + kb);
    if (rest > 0 && nrhs > 0)
      cta_gemm(rest, nrhs, kb, -1.0, LU + (k0 + kb) + size_t(k0) * lda, lda, B + k0, ldb, 1.0,
               B + k0 + kb, ldb);
  }
  // backward: upper
  for (int k1 = N; k1 > 0; k1 -= NBL) {
    const int k0 = max(0, k1 - NBL), kb = k1 - k0;
    cta_trsm_small<false>(kb, LU + k0 + size_t(k0) * lda, lda, B + k0, ldb, 0, nrhs);
    if (k0 > 0 && nrhs > 0)
      cta_gemm(k0, nrhs, kb, -1.0, LU + size_t(k0) * lda, lda, B + k0, ldb, 1.0, B, ldb);
  }
}

// Pade-13 scaling-and-squaring exponential (Higham 2005), in place on X (N x N, ld = ldx).
// work: 7 matrices of ld x N.  Returns the number of squarings.
__device__ inline int cta_expm_pade13(int N, double* X, int ldx, double* work, int ldw, int* piv,
                                      double* red, Grp g, double* psm, int psm_cap) {
  const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                        1187353796428800.0,  129060195264000.0,   10559470521600.0,
                        670442572800.0,      33522128640.0,       1323241920.0,
                        40840800.0,          960960.0,            16380.0,
                        182.0,               1.0};
  const double theta13 = 5.371920351148152;
  const size_t W = size_t(ldw) * N;
  double *A2 = work, *A4 = work + W, *A6 = work + 2 * W, *T1 = work + 3 * W, *T2 = work + 4 * W,
         *U = work + 5 * W, *V = work + 6 * W;
  double nrm = cta_norm1(N, X, ldx, red);
  int s = 0;
  if (nrm > theta13) s = max(0, (int)ceil(log2(nrm / theta13)));
  grp_sync(g);  // every CTA has read X before it is rescaled
  if (s > 0) cta_axpby(N, ldexp(1.0, -s), X, ldx, 0.0, X, ldx, 0.0, g);
  cta_gemm(N, N, N, 1.0, X, ldx, X, ldx, 0.0, A2, ldw, g);
  cta_gemm(N, N, N, 1.0, A2, ldw, A2, ldw, 0.0, A4, ldw, g);
  cta_gemm(N, N, N, 1.0, A4, ldw, A2, ldw, 0.0, A6, ldw, g);
  // U = X [A6 (b13 A6 + b11 A4 + b9 A2) + b7 A6 + b5 A4 + b3 A2 + b1 I]
  for (int idx = threadIdx.x + g.rank * blockDim.x; idx < N * N; idx += blockDim.x * g.size) {
    int i = idx % N, j = idx / N;
    size_t o = i + size_t(j) * ldw;
    T1[o] = b[13] * A6[o] + b[11] * A4[o] + b[9] * A2[o];
    T2[o] = b[7] * A6[o] + b[5] * A4[o] + b[3] * A2[o] + (i == j ? b[1] : 0.0);
  }
  grp_sync(g);
  cta_gemm(N, N, N, 1.0, A6, ldw, T1, ldw, 1.0, T2, ldw, g);
  cta_gemm(N, N, N, 1.0, X, ldx, T2, ldw, 0.0, U, ldw, g);
  // V = A6 (b12 A6 + b10 A4 + b8 A2) + b6 A6 + b4 A4 + b2 A2 + b0 I
  for (int idx = threadIdx.x + g.rank * blockDim.x; idx < N * N; idx += blockDim.x * g.size) {
    int i = idx % N, j = idx / N;
    size_t o = i + size_t(j) * ldw;
    T1[o] = b[12] * A6[o] + b[10] * A4[o] + b[8] * A2[o];
    V[o] = b[6] * A6[o] + b[4] * A4[o] + b[2] * A2[o] + (i == j ? b[0] : 0.0);
  }
  grp_sync(g);
  cta_gemm(N, N, N, 1.0, A6, ldw, T1, ldw, 1.0, V, ldw, g);
  // (V - U) R = (V + U)
  for (int idx = threadIdx.x + g.rank * blockDim.x; idx < N * N; idx += blockDim.x * g.size) {
    int i = idx % N, j = idx / N;
    size_t o = i + size_t(j) * ldw;
    T1[o] = V[o] - U[o];
    T2[o] = V[o] + U[o];
  }
  grp_sync(g);
  cta_lu(N, T1, ldw, piv, red, g, psm, psm_cap);
  cta_lu_solve(N, T1, ldw, piv, T2, ldw, N, g, psm, psm_cap);
  // squarings, ping-pong T2 <-> T1
  double *cur = T2, *nxt = T1;
  for (int q = 0; q < s; ++q) {
    cta_gemm(N, N, N, 1.0, cur, ldw, cur, ldw, 0.0, nxt, ldw, g);
    double* tmp = cur; cur = nxt; nxt = tmp;
  }
  cta_copy(N, N, cur, ldw, X, ldx, g);
  return s;
}

}  // namespace pexp
