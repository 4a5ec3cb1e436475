// tridiag.cu — subsystem (1): batched shift-and-invert solves x = (I - gamma*A)^{-1} b
// for tridiagonal (Dirichlet) and periodic-tridiagonal A (PAPER.md:176 shift-and-invert;
// DESIGN.md §5.1).
//
// Design (B200): each (operator, gamma) pair is factored ONCE per solve/WR iteration
// (Thomas LU of the tridiagonal part T plus the Sherman–Morrison vectors of the periodic
// corners, M = T + u v^T), and every Krylov right-hand side is then solved by two
// HBM-streaming passes in one CTA: the first-order recurrences of the L- and U-solves
// are affine maps y_i = a_i y_{i-1} + b_i, evaluated as a chunked block-wide parallel
// scan (8 consecutive rows per thread in registers, warp-shuffle + shared-memory scan of
// the composed maps, carry across 2048-row chunks).  The periodic correction
// x = T^{-1}b - (w'^T b) z needs only a dot product with a precomputed w' = T^{-T}v/(1+v^T z),
// accumulated during the forward pass, so no third pass is needed.
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace pexp {

// ---------------------------------------------------------------- operator rows
// A = nu*D2 - a*D1: sub = nu/dx^2 + a/(2dx), diag = -2 nu/dx^2, sup = nu/dx^2 - a/(2dx).
__global__ void k_ade_rows(int nops, int n, int dirichlet, const double* nu, const double* a,
                           double* sub, double* diag, double* sup) {
  int op = blockIdx.y;
  double dx = dirichlet ? 1.0 / (n + 1) : 1.0 / n;
  double d2 = nu[op] / (dx * dx), d1 = a[op] / (2.0 * dx);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    size_t k = size_t(op) * n + i;
    sub[k] = d2 + d1;
    diag[k] = -2.0 * d2;
    sup[k] = d2 - d1;
  }
}

// Burgers operator A_j = nu*D2 + J(ubar_j), J(u) = -diag(D1 u) - diag(u) D1 (PAPER.md:297-301,
// reading #3): sub = nu/dx^2 + ubar_i/(2dx), diag = -2nu/dx^2 - (ubar_{i+1}-ubar_{i-1})/(2dx),
// sup = nu/dx^2 - ubar_i/(2dx); periodic.
__global__ void k_burgers_rows(int nops, int n, double nu, const double* ubar, double* sub,
                               double* diag, double* sup) {
  int op = blockIdx.y;
  double dx = 1.0 / n, d2 = nu / (dx * dx), inv2dx = 1.0 / (2.0 * dx);
  const double* u = ubar + size_t(op) * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int im = i == 0 ? n - 1 : i - 1, ip = i == n - 1 ? 0 : i + 1;
    size_t k = size_t(op) * n + i;
    double ui = u[i];
    sub[k] = d2 + ui * inv2dx;
    diag[k] = -2.0 * d2 - (u[ip] - u[im]) * inv2dx;
    sup[k] = d2 - ui * inv2dx;
  }
}

// ---------------------------------------------------------------- factorisation
// One thread per factor f: M = I - gamma_f A_{op_f}.  Writes l (multipliers), dinv (1/pivot),
// msup (super-diagonal of M), and for periodic z = T^{-1}u, w' = T^{-T}v/(1+v^T z)
// with the Numerical-Recipes splitting u = (gs,0..,0,alpha), v = (1,0..,0,beta/gs), gs = -M_00.
// The recurrences are sequential; every pass reads its operands in register blocks of FCH rows
// (independent loads in flight) so that only the arithmetic dependence chain is serial.
constexpr int FCH = 16;
__global__ void k_factor(int nf, int n, int periodic, const int* __restrict__ opidx, const double* __restrict__ gam,
                         const double* __restrict__ sub, const double* __restrict__ diag,
                         const double* __restrict__ sup, double* __restrict__ fl, double* __restrict__ fdinv,
                         double* __restrict__ fsup, double* __restrict__ fz, double* __restrict__ fw,
                         int* __restrict__ err) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  const double g = gam[f];
  const size_t o = size_t(opidx ? opidx[f] : f) * n, fo = size_t(f) * n;
  const double *A = sub + o, *B = diag + o, *C = sup + o;
  double *l = fl + fo, *di = fdinv + fo, *cs = fsup + fo;
  const double d0 = 1.0 - g * B[0];
  double alpha = 0.0, beta = 0.0, gs = 0.0;
  if (periodic) {
    beta = -g * A[0];       // M[0][n-1]
    alpha = -g * C[n - 1];  // M[n-1][0]
    gs = -d0;
  }
  double dprev = periodic ? d0 - gs : d0;
  // pivots must be finite and not tiny relative to their row (no positivity needed: in the
  // cell-Peclet > 2 regime the periodic corner legitimately makes the last pivot negative)
  bool bad = !(fabs(dprev) > 1e-13 * fabs(d0)) || !isfinite(dprev);
  l[0] = 0.0;
  di[0] = 1.0 / dprev;
  double cprev = -g * C[0];
  cs[0] = cprev;
  for (int i0 = 1; i0 < n; i0 += FCH) {
    double a[FCH], bb[FCH], cc[FCH];
#pragma unroll
    for (int k = 0; k < FCH; ++k) {
      const int i = i0 + k;
      a[k] = i < n ? A[i] : 0.0;
      bb[k] = i < n ? B[i] : 0.0;
      cc[k] = i < n - 1 ? C[i] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < FCH; ++k) {
      const int i = i0 + k;
      if (i < n) {
        double Ti = 1.0 - g * bb[k];
        if (periodic && i == n - 1) Ti -= alpha * beta / gs;
        const double li = (-g * a[k]) / dprev;
        const double d = Ti - li * cprev;
        if (!(fabs(d) > 1e-13 * (fabs(Ti) + fabs(li * cprev))) || !isfinite(d)) bad = true;
        l[i] = li;
        di[i] = 1.0 / d;
        cprev = -g * cc[k];
        cs[i] = i < n - 1 ? cprev : 0.0;
        dprev = d;
      }
    }
  }
  if (periodic) {
    double *z = fz + fo, *w = fw + fo;
    // z = T^{-1} u : forward L-solve, backward U-solve
    double zp = gs;
    z[0] = gs;
    for (int i0 = 1; i0 < n; i0 += FCH) {
      double lv[FCH];
#pragma unroll
      for (int k = 0; k < FCH; ++k) lv[k] = i0 + k < n ? l[i0 + k] : 0.0;
#pragma unroll
      for (int k = 0; k < FCH; ++k)
        if (i0 + k < n) {
          zp = ((i0 + k == n - 1) ? alpha : 0.0) - lv[k] * zp;
          z[i0 + k] = zp;
        }
    }
    zp = z[n - 1] * di[n - 1];
    z[n - 1] = zp;
    for (int i1 = n - 2; i1 >= 0; i1 -= FCH) {
      double zv[FCH], cv[FCH], dv[FCH];
#pragma unroll
      for (int k = 0; k < FCH; ++k) {
        const int i = i1 - k;
        zv[k] = i >= 0 ? z[i] : 0.0;
        cv[k] = i >= 0 ? cs[i] : 0.0;
        dv[k] = i >= 0 ? di[i] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < FCH; ++k)
        if (i1 - k >= 0) {
          zp = (zv[k] - cv[k] * zp) * dv[k];
          z[i1 - k] = zp;
        }
    }
    // w = T^{-T} v :  U^T q = v, then L^T w = q
    const double vl = beta / gs;
    double wp = 1.0 * di[0];
    w[0] = wp;
    for (int i0 = 1; i0 < n; i0 += FCH) {
      double cv[FCH], dv[FCH];
#pragma unroll
      for (int k = 0; k < FCH; ++k) {
        cv[k] = i0 + k < n ? cs[i0 + k - 1] : 0.0;
        dv[k] = i0 + k < n ? di[i0 + k] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < FCH; ++k)
        if (i0 + k < n) {
          wp = (((i0 + k == n - 1) ? vl : 0.0) - cv[k] * wp) * dv[k];
          w[i0 + k] = wp;
        }
    }
    for (int i1 = n - 2; i1 >= 0; i1 -= FCH) {
      double wv[FCH], lv[FCH];
#pragma unroll
      for (int k = 0; k < FCH; ++k) {
        const int i = i1 - k;
        wv[k] = i >= 0 ? w[i] : 0.0;
        lv[k] = i >= 0 ? l[i + 1] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < FCH; ++k)
        if (i1 - k >= 0) {
          wp = wv[k] - lv[k] * wp;
          w[i1 - k] = wp;
        }
    }
    const double denom = 1.0 + z[0] + vl * z[n - 1];
    if (!(fabs(denom) > 0.0) || !isfinite(denom)) bad = true;
    const double inv = 1.0 / denom;
    for (int i = 0; i < n; ++i) w[i] *= inv;
  }
  if (bad) atomicExch(err, 1);
}

// ---------------------------------------------------------------- parallel factorisation
// One CTA per factor.  The pivot recurrence d_i = T_i - p_i / d_{i-1} (p_i = (-g a_i)(-g c_{i-1}),
// Thomas LU without pivoting) is a Moebius map of d_{i-1}: in projective coordinates
// (x, y) -> (T_i x - p_i y, x), d = x / y, i.e. a product of 2x2 matrices.  Per 2048-row tile, each
// thread composes the matrices of its 8 consecutive rows (normalised by the largest entry; the map
// is scale-free), a block-wide exclusive scan gives every thread the composed map of the rows before
// it, applied to the tile's carry-in pivot; each thread then re-runs the exact Thomas recurrence over
// its 8 rows (so l, 1/d, the superdiagonal and the pivot test are computed exactly as the sequential
// recurrence does, from a start value accurate to rounding), and the tile's last pivot is the next
// tile's carry.  The periodic Sherman-Morrison vectors z = T^{-1} u and w' = T^{-T} v / (1 + v^T z)
// are affine-map scans (forward / backward) like the shift-and-invert solve itself.
struct Mob {
  double a, b, c, d;  // [[a, b], [c, d]]
};
__device__ __forceinline__ Mob mob_then(const Mob& f, const Mob& t) {  // t * f, normalised
  Mob r{t.a * f.a + t.b * f.c, t.a * f.b + t.b * f.d, t.c * f.a + t.d * f.c, t.c * f.b + t.d * f.d};
  const double m = fmax(fmax(fabs(r.a), fabs(r.b)), fmax(fabs(r.c), fabs(r.d)));
  if (m > 0.0 && isfinite(m)) {
    const double s = 1.0 / m;
    r.a *= s; r.b *= s; r.c *= s; r.d *= s;
  }
  return r;
}

// exclusive block scan of Moebius matrices in thread order (composition: later rows on the left)
__device__ inline Mob block_excl_scan_mob(Mob v, Mob* wsm) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  Mob inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Mob p{__shfl_up_sync(0xffffffffu, inc.a, o), __shfl_up_sync(0xffffffffu, inc.b, o),
          __shfl_up_sync(0xffffffffu, inc.c, o), __shfl_up_sync(0xffffffffu, inc.d, o)};
    if (lane >= o) inc = mob_then(p, inc);
  }
  Mob exc{__shfl_up_sync(0xffffffffu, inc.a, 1), __shfl_up_sync(0xffffffffu, inc.b, 1),
          __shfl_up_sync(0xffffffffu, inc.c, 1), __shfl_up_sync(0xffffffffu, inc.d, 1)};
  if (lane == 0) exc = Mob{1.0, 0.0, 0.0, 1.0};
  __syncthreads();
  if (lane == 31) wsm[w] = inc;
  __syncthreads();
  if (t == 0) {
    Mob acc{1.0, 0.0, 0.0, 1.0};
    for (int k = 0; k < PEXP_THREADS / 32; ++k) {
      const Mob q = wsm[k];
      wsm[k] = acc;
      acc = mob_then(acc, q);
    }
  }
  __syncthreads();
  const Mob pre = wsm[w];
  __syncthreads();
  return mob_then(pre, exc);
}

// One affine first-order recurrence over all n rows, y_g = A(g) y_prev + B(g), in forward
// (rows ascending) or backward order, tile by tile with a block scan per tile; y written to out.
template <bool BWD, class FA, class FB>
__device__ inline void cta_affine_pass(int n, FA fa, FB fb, double* out, Aff* wsm) {
  const int t = threadIdx.x;
  const int nchunk = (n + CHUNK - 1) / CHUNK;
  double carry = 0.0;
  for (int q = 0; q < nchunk; ++q) {
    const int ch = BWD ? nchunk - 1 - q : q;
    const int g0 = ch * CHUNK + t * EPT;
    double av[EPT], bv[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int g = g0 + k;
      av[k] = g < n ? fa(g) : 1.0;
      bv[k] = g < n ? fb(g) : 0.0;
    }
    Aff m{1.0, 0.0};
    if (BWD) {
#pragma unroll
      for (int k = EPT - 1; k >= 0; --k) m = after(m, Aff{av[k], bv[k]});
    } else {
#pragma unroll
      for (int k = 0; k < EPT; ++k) m = after(m, Aff{av[k], bv[k]});
    }
    Aff tot;
    const Aff pre = block_excl_scan<BWD>(m, BWD ? PEXP_THREADS - 1 - t : t, wsm, tot);
    double y = fma(pre.A, carry, pre.B);
    if (BWD) {
#pragma unroll
      for (int k = EPT - 1; k >= 0; --k) {
        y = fma(av[k], y, bv[k]);
        if (g0 + k < n) out[g0 + k] = y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        y = fma(av[k], y, bv[k]);
        if (g0 + k < n) out[g0 + k] = y;
      }
    }
    carry = fma(tot.A, carry, tot.B);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(PEXP_THREADS)
k_factor_par(int n, int periodic, const int* __restrict__ opidx, const double* __restrict__ gam,
             const double* __restrict__ sub, const double* __restrict__ diag, const double* __restrict__ sup,
             double* __restrict__ fl, double* __restrict__ fdinv, double* __restrict__ fsup, double* __restrict__ fz,
             double* __restrict__ fw, int* __restrict__ err) {
  __shared__ Mob wm[PEXP_THREADS / 32];
  __shared__ Aff wsm[PEXP_THREADS / 32 + 1];
  __shared__ double s_carry;
  __shared__ int s_bad;
  const int f = blockIdx.x, t = threadIdx.x;
  const double g = gam[f];
  const size_t o = size_t(opidx ? opidx[f] : f) * n, fo = size_t(f) * n;
  const double *A = sub + o, *B = diag + o, *C = sup + o;
  double *l = fl + fo, *di = fdinv + fo, *cs = fsup + fo;
  const double d0 = 1.0 - g * B[0];
  double alpha = 0.0, beta = 0.0, gs = 0.0;
  if (periodic) {
    beta = -g * A[0];       // M[0][n-1]
    alpha = -g * C[n - 1];  // M[n-1][0]
    gs = -d0;
  }
  const double dfirst = periodic ? d0 - gs : d0;
  if (t == 0) {
    s_carry = dfirst;
    s_bad = !(fabs(dfirst) > 1e-13 * fabs(d0)) || !isfinite(dfirst);
  }
  __syncthreads();
  bool bad = false;
  auto Tdiag = [&](int i) {
    double Ti = 1.0 - g * B[i];
    if (periodic && i == n - 1) Ti -= alpha * beta / gs;
    return Ti;
  };
  const int nchunk = (n + CHUNK - 1) / CHUNK;
  for (int ch = 0; ch < nchunk; ++ch) {
    const int g0 = ch * CHUNK + t * EPT;
    double Tv[EPT], av[EPT], cp[EPT];  // T_i, -g a_i, -g c_{i-1}
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = g0 + k;
      const bool ok = i >= 1 && i < n;
      Tv[k] = ok ? Tdiag(i) : 1.0;
      av[k] = ok ? -g * A[i] : 0.0;
      cp[k] = ok ? -g * C[i - 1] : 0.0;
    }
    Mob m{1.0, 0.0, 0.0, 1.0};  // row 0 and rows >= n: identity (row 0's pivot is the carry-in)
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (g0 + k >= 1 && g0 + k < n) m = mob_then(m, Mob{Tv[k], -av[k] * cp[k], 1.0, 0.0});
    const Mob pre = block_excl_scan_mob(m, wm);
    const double c0 = s_carry;  // pivot of the row before this tile (row 0's pivot for tile 0)
    const double x = pre.a * c0 + pre.b, y = pre.c * c0 + pre.d;
    double dprev = x / y;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int i = g0 + k;
      if (i == 0) {
        l[0] = 0.0;
        di[0] = 1.0 / dfirst;
        cs[0] = -g * C[0];
        dprev = dfirst;
      } else if (i < n) {
        const double li = av[k] / dprev;
        const double d = Tv[k] - li * cp[k];
        if (!(fabs(d) > 1e-13 * (fabs(Tv[k]) + fabs(li * cp[k]))) || !isfinite(d)) bad = true;
        l[i] = li;
        di[i] = 1.0 / d;
        cs[i] = i < n - 1 ? -g * C[i] : 0.0;
        dprev = d;
      }
    }
    __syncthreads();                            // every thread has read s_carry
    if (t == PEXP_THREADS - 1) s_carry = dprev;  // last row of a full tile: the next tile's carry
    __syncthreads();
  }
  if (bad) s_bad = 1;
  __syncthreads();
  if (periodic) {
    double *z = fz + fo, *w = fw + fo;
    __syncthreads();
    // z = T^{-1} u, u = (gs, 0, .., 0, alpha): y_i = u_i - l_i y_{i-1}; z_i = d_i^{-1} (y_i - cs_i z_{i+1})
    cta_affine_pass<false>(
        n, [&](int i) { return -l[i]; },
        [&](int i) { return i == 0 ? gs : (i == n - 1 ? alpha : 0.0); }, z, wsm);
    __syncthreads();
    cta_affine_pass<true>(
        n, [&](int i) { return -di[i] * cs[i]; }, [&](int i) { return di[i] * z[i]; }, z, wsm);
    __syncthreads();
    // w = T^{-T} v, v = (1, 0, .., 0, beta/gs): U^T q = v, then L^T w = q
    const double vl = beta / gs;
    cta_affine_pass<false>(
        n, [&](int i) { return i == 0 ? 0.0 : -di[i] * cs[i - 1]; },
        [&](int i) { return di[i] * (i == 0 ? 1.0 : (i == n - 1 ? vl : 0.0)); }, w, wsm);
    __syncthreads();
    cta_affine_pass<true>(
        n, [&](int i) { return i == n - 1 ? 0.0 : -l[i + 1]; }, [&](int i) { return w[i]; }, w, wsm);
    __syncthreads();
    const double denom = 1.0 + z[0] + vl * z[n - 1];
    if (!(fabs(denom) > 0.0) || !isfinite(denom)) bad = true;
    const double inv = 1.0 / denom;
    for (int i = t; i < n; i += PEXP_THREADS) w[i] *= inv;
    if (bad) s_bad = 1;
    __syncthreads();
  }
  if (t == 0 && s_bad) atomicExch(err, 1);
}

// Grid (ncols, E).  Column c of eval e: rhs at rhs + e*rs_e + (cin0+c)*n, result at
// out + e*os_e + (cout0+c)*n (may alias rhs only if identical).  fidx[e] selects the factor.
__global__ void __launch_bounds__(PEXP_THREADS, 2)
k_sai_solve(int n, int periodic, const int* fidx, const double* fl, const double* fdinv,
            const double* fsup, const double* fz, const double* fw, const double* rhs,
            long long rs_e, int cin0, double* out, long long os_e, int cout0,
            const int* active, double* out2, long long o2s_e) {
  const int c = blockIdx.x, e = blockIdx.y;
  if (active && !active[e]) return;
  __shared__ double s0[PEXP_THREADS * SPAD];
  __shared__ double s1[PEXP_THREADS * SPAD];
  __shared__ Aff wsm[PEXP_THREADS / 32 + 1];
  __shared__ double red[32];
  const size_t fo = size_t(fidx ? fidx[e] : e) * n;
  cta_sai_solve(n, periodic, fl + fo, fdinv + fo, fsup + fo, periodic ? fz + fo : nullptr, periodic ? fw + fo : nullptr,
                rhs + e * rs_e + size_t(cin0 + c) * n, out + e * os_e + size_t(cout0 + c) * n,
                out2 ? out2 + e * o2s_e + size_t(c) * n : nullptr, s0, s1, wsm, red);
}

// ---------------------------------------------------------------- host wrappers
void launch_ade_rows(cudaStream_t st, int nops, int n, bool dirichlet, const double* nu,
                     const double* a, double* sub, double* diag, double* sup) {
  dim3 grid(std::min(cdiv(n, PEXP_THREADS), 64), nops);
  k_ade_rows<<<grid, PEXP_THREADS, 0, st>>>(nops, n, dirichlet ? 1 : 0, nu, a, sub, diag, sup);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_burgers_rows(cudaStream_t st, int nops, int n, double nu, const double* ubar,
                         double* sub, double* diag, double* sup) {
  dim3 grid(std::min(cdiv(n, PEXP_THREADS), 64), nops);
  k_burgers_rows<<<grid, PEXP_THREADS, 0, st>>>(nops, n, nu, ubar, sub, diag, sup);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_factor(cudaStream_t st, const Factors& F, int nf, const int* opidx, const double* gam,
                   const Ops& O, int* err) {
  ProfScope ps(PC_FACTOR, st, double(nf) * F.n * 8.0 * (3 + 3 + (F.periodic ? 2 : 0)), 0.0);
  if (F.n >= CHUNK)  // long columns: one CTA per factor, block scans (k_factor_par)
    k_factor_par<<<nf, PEXP_THREADS, 0, st>>>(F.n, F.periodic, opidx, gam, O.sub, O.diag, O.sup, F.l, F.dinv, F.sup,
                                              F.z, F.w, err);
  else
    k_factor<<<cdiv(nf, 64), 64, 0, st>>>(nf, F.n, F.periodic, opidx, gam, O.sub, O.diag, O.sup, F.l, F.dinv, F.sup,
                                          F.z, F.w, err);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_sai_solve(cudaStream_t st, const Factors& F, const int* fidx, int E, int ncols,
                      const double* rhs, long long rs_e, int cin0, double* out, long long os_e,
                      int cout0, const int* active, double* out2, long long o2s_e) {
  if (E == 0 || ncols == 0) return;
  // algorithmic: read rhs + write x per column, factors once per distinct factor (<= E)
  const double ea = eact(E, active);
  ProfScope ps(PC_SOLVE, st, ea * ncols * F.n * 16.0 + std::min(ea, double(F.nf)) * F.n * 8.0 * (F.periodic ? 5 : 3),
               ea * ncols * F.n * (F.periodic ? 8.0 : 6.0));
  dim3 grid(ncols, E);
  k_sai_solve<<<grid, PEXP_THREADS, 0, st>>>(F.n, F.periodic, fidx, F.l, F.dinv, F.sup, F.z, F.w,
                                              rhs, rs_e, cin0, out, os_e, cout0, active, out2, o2s_e);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

}  // namespace pexp
