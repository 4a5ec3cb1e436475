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

// Grid (ncols, E).  Column c of eval e: rhs at rhs + e*rs_e + (cin0+c)*n, result at
// out + e*os_e + (cout0+c)*n (may alias rhs only if identical).  fidx[e] selects the factor.
__global__ void __launch_bounds__(PEXP_THREADS)
k_sai_solve(int n, int periodic, const int* fidx, const double* fl, const double* fdinv,
            const double* fsup, const double* fz, const double* fw, const double* rhs,
            long long rs_e, int cin0, double* out, long long os_e, int cout0,
            const int* active) {
  const int c = blockIdx.x, e = blockIdx.y;
  if (active && !active[e]) return;
  __shared__ double s0[PEXP_THREADS * SPAD];
  __shared__ double s1[PEXP_THREADS * SPAD];
  __shared__ Aff wsm[PEXP_THREADS / 32 + 1];
  __shared__ double red[32];
  const size_t fo = size_t(fidx ? fidx[e] : e) * n;
  cta_sai_solve(n, periodic, fl + fo, fdinv + fo, fsup + fo, periodic ? fz + fo : nullptr, periodic ? fw + fo : nullptr,
                rhs + e * rs_e + size_t(cin0 + c) * n, out + e * os_e + size_t(cout0 + c) * n, nullptr, s0, s1, wsm,
                red);
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
  k_factor<<<cdiv(nf, 64), 64, 0, st>>>(nf, F.n, F.periodic, opidx, gam, O.sub, O.diag, O.sup,
                                         F.l, F.dinv, F.sup, F.z, F.w, err);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_sai_solve(cudaStream_t st, const Factors& F, const int* fidx, int E, int ncols,
                      const double* rhs, long long rs_e, int cin0, double* out, long long os_e,
                      int cout0, const int* active) {
  if (E == 0 || ncols == 0) return;
  // algorithmic: read rhs + write x per column, factors once per distinct factor (<= E)
  const double ea = eact(E, active);
  ProfScope ps(PC_SOLVE, st, ea * ncols * F.n * 16.0 + std::min(ea, double(F.nf)) * F.n * 8.0 * (F.periodic ? 5 : 3),
               ea * ncols * F.n * (F.periodic ? 8.0 : 6.0));
  dim3 grid(ncols, E);
  k_sai_solve<<<grid, PEXP_THREADS, 0, st>>>(F.n, F.periodic, fidx, F.l, F.dinv, F.sup, F.z, F.w,
                                              rhs, rs_e, cin0, out, os_e, cout0, active);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

}  // namespace pexp
