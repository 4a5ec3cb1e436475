// scan.cuh — CTA-wide affine-map scans and the per-column shift-and-invert solve
// (subsystem 1) shared by k_sai_solve (tridiag.cu) and the fused Arnoldi step (arnoldi.cu).
#pragma once
#include "common.cuh"

namespace pexp {

// ---------------------------------------------------------------- affine-map block scan
// Map f(y) = A*y + B.  compose(first, then) = then ∘ first.
struct Aff {
  double A, B;
};
__device__ __forceinline__ Aff after(Aff first, Aff then) {
  return {then.A * first.A, fma(then.A, first.B, then.B)};
}

// Exclusive scan over the block (ordered by `rank`, 0..255) of the per-thread maps.
// rank = threadIdx.x (forward) or 255 - threadIdx.x (reverse, REV = true); in the reverse
// order the lane of rank-predecessor k-o is the PHYSICAL lane +o, hence shfl_down.
// Returns the composition of all maps of lower rank (identity for rank 0) and, through
// `total`, the composition of all 256.
template <bool REV>
__device__ __forceinline__ Aff block_excl_scan(Aff v, int rank, Aff* wsm, Aff& total) {
  const int lane = rank & 31, w = rank >> 5;
  Aff inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double pa = REV ? __shfl_down_sync(0xffffffffu, inc.A, o) : __shfl_up_sync(0xffffffffu, inc.A, o);
    double pb = REV ? __shfl_down_sync(0xffffffffu, inc.B, o) : __shfl_up_sync(0xffffffffu, inc.B, o);
    if (lane >= o) inc = after(Aff{pa, pb}, inc);
  }
  double ea = REV ? __shfl_down_sync(0xffffffffu, inc.A, 1) : __shfl_up_sync(0xffffffffu, inc.A, 1);
  double eb = REV ? __shfl_down_sync(0xffffffffu, inc.B, 1) : __shfl_up_sync(0xffffffffu, inc.B, 1);
  Aff exc = lane == 0 ? Aff{1.0, 0.0} : Aff{ea, eb};
  __syncthreads();
  if (lane == 31) wsm[w] = inc;
  __syncthreads();
  if (rank == 0) {
    Aff acc{1.0, 0.0};
    for (int k = 0; k < PEXP_THREADS / 32; ++k) {
      Aff t = wsm[k];
      wsm[k] = acc;  // exclusive prefix of warp k
      acc = after(acc, t);
    }
    wsm[PEXP_THREADS / 32] = acc;
  }
  __syncthreads();
  Aff pre = wsm[w];
  total = wsm[PEXP_THREADS / 32];
  return after(pre, exc);
}

constexpr int EPT = 8;                       // rows per thread per chunk
constexpr int CHUNK = EPT * PEXP_THREADS;    // 2048 rows
constexpr int SPAD = EPT + 1;                // smem row padding (bank spread)

// Solve one column x = (I - gamma A)^{-1} b with the factor (l, di, cs, [fz, fw]) by the two
// streaming affine scans (forward L-solve, backward U-solve; periodic Sherman-Morrison correction
// through the precomputed w').  All PEXP_THREADS threads call it.  Optional copy to x2; returns
// ||x||^2 (block-reduced, valid in every thread).  s0, s1: PEXP_THREADS*SPAD doubles each.
__device__ inline double cta_sai_solve(int n, int periodic, const double* l, const double* di, const double* cs,
                                       const double* fz, const double* fw, const double* b, double* x, double* x2,
                                       double* s0, double* s1, Aff* wsm, double* red) {
  const int t = threadIdx.x;
  const int nchunk = (n + CHUNK - 1) / CHUNK;
  double carry = 0.0, dot = 0.0;
  // Software pipeline: the operands of the next chunk are loaded into registers while this chunk is
  // scanned, so the dependent chain of chunks never waits on a DRAM round trip (ncu before:
  // 48 % of the stall samples on the x / fz loads of the backward pass, profiles/r02_ncu_c5_sai_solve.txt).
  {
    double pb[EPT], pl[EPT], pw[EPT];
    auto load_fwd = [&](int ch) {
      const int base = ch * CHUNK;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int g = base + t + k * PEXP_THREADS;
        const bool ok = g < n;
        pb[k] = ok ? b[g] : 0.0;
        pl[k] = ok ? -l[g] : 1.0;
        pw[k] = (periodic && ok) ? fw[g] : 0.0;
      }
    };
    load_fwd(0);
    for (int ch = 0; ch < nchunk; ++ch) {
      const int base = ch * CHUNK;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int i = t + k * PEXP_THREADS;
        const int si = (i / EPT) * SPAD + (i % EPT);
        s0[si] = pb[k];
        s1[si] = pl[k];
        if (periodic) dot = fma(pw[k], pb[k], dot);
      }
      __syncthreads();
      if (ch + 1 < nchunk) load_fwd(ch + 1);
      Aff m{1.0, 0.0};
#pragma unroll
      for (int k = 0; k < EPT; ++k) m = after(m, Aff{s1[t * SPAD + k], s0[t * SPAD + k]});
      Aff tot;
      Aff pre = block_excl_scan<false>(m, t, wsm, tot);
      double y = fma(pre.A, carry, pre.B);
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        y = fma(s1[t * SPAD + k], y, s0[t * SPAD + k]);
        s0[t * SPAD + k] = y;
      }
      carry = fma(tot.A, carry, tot.B);
      __syncthreads();
      for (int i = t; i < CHUNK; i += PEXP_THREADS) {
        int g = base + i;
        if (g < n) x[g] = s0[(i / EPT) * SPAD + (i % EPT)];
      }
      __syncthreads();
    }
  }
  double f = 0.0;
  if (periodic) f = block_sum(dot, red);
  carry = 0.0;
  double nrm2 = 0.0;
  const int r = PEXP_THREADS - 1 - t;
  double px[EPT], pd[EPT], pc[EPT], pz[EPT];
  // x[g] of a chunk was written by this same thread in the forward pass (same row -> thread map)
  auto load_bwd = [&](int ch) {
    const int base = ch * CHUNK;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int g = base + t + k * PEXP_THREADS;
      const bool ok = g < n;
      pd[k] = ok ? di[g] : 0.0;
      px[k] = ok ? x[g] : 0.0;
      pc[k] = ok ? cs[g] : 0.0;
      pz[k] = (periodic && ok) ? fz[g] : 0.0;
    }
  };
  load_bwd(nchunk - 1);
  for (int ch = nchunk - 1; ch >= 0; --ch) {
    const int base = ch * CHUNK;
    double cz[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = t + k * PEXP_THREADS;
      const int si = (i / EPT) * SPAD + (i % EPT);
      const bool ok = base + i < n;
      s0[si] = ok ? pd[k] * px[k] : 0.0;
      s1[si] = ok ? -pd[k] * pc[k] : 1.0;
      cz[k] = pz[k];
    }
    __syncthreads();
    if (ch > 0) load_bwd(ch - 1);
    Aff m{1.0, 0.0};
#pragma unroll
    for (int k = EPT - 1; k >= 0; --k) m = after(m, Aff{s1[t * SPAD + k], s0[t * SPAD + k]});
    Aff tot;
    Aff pre = block_excl_scan<true>(m, r, wsm, tot);
    double y = fma(pre.A, carry, pre.B);
#pragma unroll
    for (int k = EPT - 1; k >= 0; --k) {
      y = fma(s1[t * SPAD + k], y, s0[t * SPAD + k]);
      s0[t * SPAD + k] = y;
    }
    carry = fma(tot.A, carry, tot.B);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = t + k * PEXP_THREADS;
      const int g = base + i;
      if (g < n) {
        double v = s0[(i / EPT) * SPAD + (i % EPT)];
        if (periodic) v = fma(-f, cz[k], v);
        x[g] = v;
        if (x2) x2[g] = v;
        nrm2 = fma(v, v, nrm2);
      }
    }
    __syncthreads();
  }
  return block_sum(nrm2, red);
}

}  // namespace pexp
