// tsmm.cu — tall-skinny fp64 products used by subsystems (2) and (3):
//   * xty:     T_e = X_e^T Y_e  (X_e: n x nx, Y_e: n x ny column slices of per-eval
//              column-major panels), split over row chunks; per-chunk partials reduced
//              deterministically by k_reduce.  Used for the block classical Gram–Schmidt
//              projections V^T W (BCGS2), block Gram matrices W^T W (CholQR2) and the
//              source Gram / cross products of the two-pass SVD.
//   * combine: Out_e = beta*Out_e + alpha * X_e M_e (n x nx times nx x ny), one thread per
//              row so that Out may alias X (in-place right-multiplication, ny <= 32).
// Loads are coalesced along rows (each warp reads 32 consecutive rows of a column);
// per-thread 4x4 register tiles accumulate the small products from shared memory.
#include <cstdlib>
#include "common.cuh"
#include "kernels.cuh"

namespace pexp {

constexpr int TR = 16;  // rows per shared-memory stage

// fp64 tensor-core MMA: D(8x8) += A(8x4, row) B(4x8, col); per lane A[lane/4][lane%4],
// B[lane%4][lane/4], D[lane/4][2(lane%4) + {0,1}]
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
constexpr int RA = 4, RB = 4;

template <int NT>
__global__ void __launch_bounds__(PEXP_THREADS)
k_xty_partial(int n, int rch, const double* X, long long xs_e, int x0, int nx, const double* Y,
              long long ys_e, int y0, int ny, double* part, const int* active) {
  extern __shared__ double sm[];
  const int e = blockIdx.y, ch = blockIdx.x, nch = gridDim.x;
  if (active && !active[e]) return;
  const int nxp = ((nx + RA - 1) / RA) * RA, nyp = ((ny + RB - 1) / RB) * RB;
  double* Xs = sm;              // [TR][nxp]
  double* Ys = sm + TR * nxp;   // [TR][nyp]
  const double* Xe = X + e * xs_e + size_t(x0) * n;
  const double* Ye = Y + e * ys_e + size_t(y0) * n;
  const int ntb = nyp / RB, ntiles = (nxp / RA) * ntb;
  double acc[NT][RA][RB];
#pragma unroll
  for (int q = 0; q < NT; ++q)
#pragma unroll
    for (int i = 0; i < RA; ++i)
#pragma unroll
      for (int j = 0; j < RB; ++j) acc[q][i][j] = 0.0;
  const int r0 = ch * rch, r1 = min(n, r0 + rch);
  for (int rb = r0; rb < r1; rb += TR) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < TR * nxp; idx += PEXP_THREADS) {
      int a = idx / TR, r = idx % TR, row = rb + r;
      Xs[r * nxp + a] = (a < nx && row < r1) ? Xe[size_t(a) * n + row] : 0.0;
    }
    for (int idx = threadIdx.x; idx < TR * nyp; idx += PEXP_THREADS) {
      int b = idx / TR, r = idx % TR, row = rb + r;
      Ys[r * nyp + b] = (b < ny && row < r1) ? Ye[size_t(b) * n + row] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      int tile = threadIdx.x + q * PEXP_THREADS;
      if (tile < ntiles) {
        int ta = tile / ntb, tb = tile % ntb;
        for (int r = 0; r < TR; ++r) {
          double xv[RA], yv[RB];
#pragma unroll
          for (int i = 0; i < RA; ++i) xv[i] = Xs[r * nxp + ta * RA + i];
#pragma unroll
          for (int j = 0; j < RB; ++j) yv[j] = Ys[r * nyp + tb * RB + j];
#pragma unroll
          for (int i = 0; i < RA; ++i)
#pragma unroll
            for (int j = 0; j < RB; ++j) acc[q][i][j] = fma(xv[i], yv[j], acc[q][i][j]);
        }
      }
    }
  }
  double* P = part + (size_t(e) * nch + ch) * size_t(nx) * ny;
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    int tile = threadIdx.x + q * PEXP_THREADS;
    if (tile < ntiles) {
      int ta = tile / ntb, tb = tile % ntb;
#pragma unroll
      for (int i = 0; i < RA; ++i)
#pragma unroll
        for (int j = 0; j < RB; ++j) {
          int a = ta * RA + i, b = tb * RB + j;
          if (a < nx && b < ny) P[a + size_t(b) * nx] = acc[q][i][j];
        }
    }
  }
}

// Tall-skinny X^T Y for ny <= 32 (the BCGS projections V^T W and block Grams): the CTA's
// row chunk of Y is staged once in shared memory (column-major, conflict-free); every warp
// streams whole X columns of the chunk (coalesced 256-B loads, 4 rows per lane in flight),
// accumulates the ny dot products per lane and reduces them with warp shuffles.  X is read
// exactly once from HBM; Y once per chunk.
// Deterministic fused split-K reduction: every CTA publishes its partial, the LAST CTA of the
// evaluation (ticket counter) sums the partials in chunk order and writes D; the counter is
// reset for the next launch.
struct RedArgs {
  double* D;
  long long ds_e;
  int ldd, row0, col0, accumulate;
  int* cnt;  // [E] zero-initialised tickets (nullptr: separate k_reduce launch)
};

__device__ __forceinline__ void last_cta_reduce(const RedArgs& ra, const double* part, int e, int nch, int nx,
                                                int ny) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ra.cnt + e, 1) == nch - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const size_t sz = size_t(nx) * ny;
  const double* pe = part + size_t(e) * nch * sz;
  for (int idx = threadIdx.x; idx < nx * ny; idx += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < nch; ++c) acc += __ldcg(pe + c * sz + idx);
    int a = idx % nx, b = idx / nx;
    double* d = ra.D + e * ra.ds_e + (ra.row0 + a) + size_t(ra.col0 + b) * ra.ldd;
    *d = ra.accumulate ? *d + acc : acc;
  }
  if (threadIdx.x == 0) ra.cnt[e] = 0;
}

template <int NYB>
__global__ void __launch_bounds__(PEXP_THREADS)
k_xty_tall(int n, int rch, int rsub, const double* X, long long xs_e, int x0, int nx, const double* Y, long long ys_e,
           int y0, int ny, double* part, const int* active, RedArgs ra) {
  extern __shared__ double sm[];
  double* Ys = sm;                 // [ny][rsub]   current sub-chunk of Y (column-major)
  double* Ps = sm + ny * rsub;     // [nx][ny]     CTA partial
  const int e = blockIdx.y, ch = blockIdx.x, nch = gridDim.x;
  if (active && !active[e]) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = PEXP_THREADS / 32;
  for (int i = threadIdx.x; i < nx * ny; i += PEXP_THREADS) Ps[i] = 0.0;
  const int cbeg = ch * rch, cend = min(n, cbeg + rch);
  for (int r0 = cbeg; r0 < cend; r0 += rsub) {
    const int rows = min(rsub, cend - r0);
    const double* Xe = X + e * xs_e + size_t(x0) * n + r0;
    const double* Ye = Y + e * ys_e + size_t(y0) * n + r0;
    __syncthreads();
    for (int b = 0; b < ny; ++b)
      for (int r = threadIdx.x; r < rsub; r += PEXP_THREADS) Ys[b * rsub + r] = r < rows ? Ye[size_t(b) * n + r] : 0.0;
    __syncthreads();
    for (int a = warp; a < nx; a += nw) {
      const double* xc = Xe + size_t(a) * n;
      double acc[NYB];
#pragma unroll
      for (int b = 0; b < NYB; ++b) acc[b] = 0.0;
      int r = lane;
      for (; r + 96 < rows; r += 128) {
        double x0v = xc[r], x1v = xc[r + 32], x2v = xc[r + 64], x3v = xc[r + 96];
#pragma unroll
        for (int b = 0; b < NYB; ++b) {
          if (b < ny) {
            const double* yb = Ys + b * rsub + r;
            acc[b] = fma(x0v, yb[0], acc[b]);
            acc[b] = fma(x1v, yb[32], acc[b]);
            acc[b] = fma(x2v, yb[64], acc[b]);
            acc[b] = fma(x3v, yb[96], acc[b]);
          }
        }
      }
      for (; r < rows; r += 32) {
        double xv = xc[r];
#pragma unroll
        for (int b = 0; b < NYB; ++b)
          if (b < ny) acc[b] = fma(xv, Ys[b * rsub + r], acc[b]);
      }
#pragma unroll
      for (int b = 0; b < NYB; ++b) {
        if (b < ny) {
          double v = warp_sum(acc[b]);
          if (lane == 0) Ps[a + b * nx] += v;  // column a is owned by this warp: no race
        }
      }
    }
  }
  __syncthreads();
  double* P = part + (size_t(e) * nch + ch) * size_t(nx) * ny;
  for (int i = threadIdx.x; i < nx * ny; i += PEXP_THREADS) P[i] = Ps[i];
  if (ra.cnt) last_cta_reduce(ra, part, e, nch, nx, ny);
}

// D_e[row0 + a, col0 + b] (= or +=) sum_ch part[e][ch][a + b*nx]
__global__ void k_reduce(int nx, int ny, int nch, const double* part, double* D, long long ds_e,
                         int ldd, int row0, int col0, int accumulate, const int* active) {
  const int e = blockIdx.y;
  if (active && !active[e]) return;
  const size_t sz = size_t(nx) * ny;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nx * ny; idx += gridDim.x * blockDim.x) {
    const double* p = part + size_t(e) * nch * sz + idx;
    double s = 0.0;
    for (int c = 0; c < nch; ++c) s += p[c * sz];
    int a = idx % nx, b = idx / nx;
    double* d = D + e * ds_e + (row0 + a) + size_t(col0 + b) * ldd;
    *d = accumulate ? *d + s : s;
  }
}

// Square-ish X^T Y for 32 < nx, ny <= 64 (the s x s Grams and cross products of the two-pass
// source SVD, s = 64): a stage of SQ_TR rows of X and Y sits in shared memory row-major; the
// 256 threads form 4 row groups x (8 x 8) threads, each thread owning an 8 x 8 output tile
// (4 FMA per shared load, double2 loads); the next stage is prefetched into registers while the
// current one is consumed; the 4 row-group partials are summed at the end (stage buffers reused).
constexpr int SQ_TR = 32;
__global__ void __launch_bounds__(PEXP_THREADS)
k_xty_sq(int n, int rch, const double* X, long long xs_e, int x0, int nx, const double* Y, long long ys_e, int y0,
         int ny, double* part) {
  __shared__ __align__(16) double stg[2 * SQ_TR * 64];  // Xs | Ys, later the row-group partials
  double (*Xs)[64] = reinterpret_cast<double (*)[64]>(stg);
  double (*Ys)[64] = reinterpret_cast<double (*)[64]>(stg + SQ_TR * 64);
  const int e = blockIdx.y, ch = blockIdx.x, nch = gridDim.x;
  const int t = threadIdx.x, grp = t >> 6, tx = t & 7, ty = (t >> 3) & 7;
  const double* Xe = X + e * xs_e + size_t(x0) * n;
  const double* Ye = Y + e * ys_e + size_t(y0) * n;
  const bool same = (Xe == Ye) && nx == ny;
  constexpr int LPT = SQ_TR * 64 / PEXP_THREADS;  // elements per thread per operand and stage
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  const int r0 = ch * rch, r1 = min(n, r0 + rch);
  double px[LPT], py[LPT];
  auto fetch = [&](int rb) {
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int idx = t + q * PEXP_THREADS, a = idx / SQ_TR, r = idx % SQ_TR, row = rb + r;  // rows fastest
      px[q] = (a < nx && row < r1) ? __ldcg(Xe + size_t(a) * n + row) : 0.0;
      py[q] = (!same && a < ny && row < r1) ? __ldcg(Ye + size_t(a) * n + row) : 0.0;
    }
  };
  if (r0 < r1) fetch(r0);
  for (int rb = r0; rb < r1; rb += SQ_TR) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int idx = t + q * PEXP_THREADS, a = idx / SQ_TR, r = idx % SQ_TR;
      Xs[r][a] = px[q];
      if (!same) Ys[r][a] = py[q];
    }
    __syncthreads();
    if (rb + SQ_TR < r1) fetch(rb + SQ_TR);
    const double (*Yr)[64] = same ? Xs : Ys;
#pragma unroll 2
    for (int r = grp; r < SQ_TR; r += 4) {
      double xv[8], yv[8];
      const double2* xp = reinterpret_cast<const double2*>(&Xs[r][ty * 8]);
      const double2* yp = reinterpret_cast<const double2*>(&Yr[r][tx * 8]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 a2 = xp[q], b2 = yp[q];
        xv[2 * q] = a2.x; xv[2 * q + 1] = a2.y;
        yv[2 * q] = b2.x; yv[2 * q + 1] = b2.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(xv[i], yv[j], acc[i][j]);
    }
  }
  // sum the 4 row-group partials, a quarter of every thread tile at a time (3 x 1024 doubles)
  double* red = stg;
  double* P = part + (size_t(e) * nch + ch) * size_t(nx) * ny;
#pragma unroll
  for (int qt = 0; qt < 4; ++qt) {  // rows i in [2qt, 2qt+2) of every thread tile
    __syncthreads();
    if (grp > 0)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) red[(grp - 1) * 1024 + ((ty * 2 + i) * 8 + tx) * 8 + j] = acc[2 * qt + i][j];
    __syncthreads();
    if (grp == 0)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = ((ty * 2 + i) * 8 + tx) * 8 + j;
          const double v = acc[2 * qt + i][j] + red[k] + red[1024 + k] + red[2048 + k];
          const int a = ty * 8 + 2 * qt + i, b = tx * 8 + j;
          if (a < nx && b < ny) P[a + size_t(b) * nx] = v;
        }
  }
}

constexpr int NB = 32;  // max output columns per combine launch

template <int NBT>
__global__ void __launch_bounds__(PEXP_THREADS)
k_combine(int n, const double* X, long long xs_e, int x0, int nx, const double* M, long long ms_e,
          int ldm, double* O, long long os_e, int o0, int ny, double alpha, double beta,
          const int* active, const int* nxe) {
  extern __shared__ __align__(16) double Ms[];  // [nx][NBT]
  const int e = blockIdx.y;
  if (active && !active[e]) return;
  const double* Me = M + e * ms_e;
  for (int idx = threadIdx.x; idx < nx * NBT; idx += PEXP_THREADS) {
    int a = idx / NBT, b = idx % NBT;
    Ms[idx] = b < ny ? Me[a + size_t(b) * ldm] : 0.0;
  }
  __syncthreads();
  // two rows per thread (r, r + 256): every shared-memory value feeds two FMAs, read as double2
  const int row = blockIdx.x * (2 * PEXP_THREADS) + threadIdx.x;
  if (row >= n) return;
  const bool two = row + PEXP_THREADS < n;
  const double* Xe = X + e * xs_e + size_t(x0) * n + row;
  const int nxl = nxe ? min(nx, nxe[e]) : nx;
  double acc0[NBT], acc1[NBT];
#pragma unroll
  for (int b = 0; b < NBT; ++b) { acc0[b] = 0.0; acc1[b] = 0.0; }
  int a = 0;
  for (; a + 3 < nxl; a += 4) {  // 4 columns x 2 rows of independent loads in flight
    double x0v[4], x1v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0v[u] = __ldcg(Xe + size_t(a + u) * n);
      x1v[u] = two ? __ldcg(Xe + size_t(a + u) * n + PEXP_THREADS) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2* mr = reinterpret_cast<const double2*>(Ms + (a + u) * NBT);
#pragma unroll
      for (int b = 0; b < NBT / 2; ++b) {
        const double2 mv = mr[b];
        acc0[2 * b] = fma(x0v[u], mv.x, acc0[2 * b]);
        acc0[2 * b + 1] = fma(x0v[u], mv.y, acc0[2 * b + 1]);
        acc1[2 * b] = fma(x1v[u], mv.x, acc1[2 * b]);
        acc1[2 * b + 1] = fma(x1v[u], mv.y, acc1[2 * b + 1]);
      }
    }
  }
  for (; a < nxl; ++a) {
    const double xv = Xe[size_t(a) * n], xw = two ? Xe[size_t(a) * n + PEXP_THREADS] : 0.0;
    const double* mr = Ms + a * NBT;
#pragma unroll
    for (int b = 0; b < NBT; ++b) {
      acc0[b] = fma(xv, mr[b], acc0[b]);
      acc1[b] = fma(xw, mr[b], acc1[b]);
    }
  }
  double* Oe = O + e * os_e + size_t(o0) * n + row;
#pragma unroll
  for (int b = 0; b < NBT; ++b)
    if (b < ny) {
      double v = alpha * acc0[b];
      if (beta != 0.0) v = fma(beta, Oe[size_t(b) * n], v);
      Oe[size_t(b) * n] = v;
      if (two) {
        double w = alpha * acc1[b];
        if (beta != 0.0) w = fma(beta, Oe[size_t(b) * n + PEXP_THREADS], w);
        Oe[size_t(b) * n + PEXP_THREADS] = w;
      }
    }
}

// Tall-skinny X^T Y on the fp64 tensor cores for the large projections (nx >= 32, 8 < ny <= 32):
// grid (row chunks, 64-column blocks of X, E).  Per 16-row step the CTA stages X (16 x 64) and
// Y (16 x NYT) in shared memory (next step prefetched into registers); warp w owns the m8 tile w
// of the 64 X columns and all NYT/8 n8 tiles (DMMA m8n8k4).  Partials per chunk, reduced by k_reduce.
template <int NYT>
__global__ void __launch_bounds__(PEXP_THREADS)
k_xty_mma(int n, int rch, const double* X, long long xs_e, int x0, int nx, const double* Y, long long ys_e, int y0,
          int ny, double* part, const int* active) {
  constexpr int XC = 64, LDX = XC + 8, LDY = NYT + 8, NJ = NYT / 8;
  constexpr int LX = 16 * XC / PEXP_THREADS, LY = (16 * NYT + PEXP_THREADS - 1) / PEXP_THREADS;
  __shared__ __align__(16) double Xs[16][LDX];
  __shared__ __align__(16) double Ys[16][LDY];
  const int ch = blockIdx.x, cb = blockIdx.y, e = blockIdx.z, nch = gridDim.x;
  if (active && !active[e]) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, fr = lane >> 2, fc = lane & 3;
  const int a0 = cb * XC;
  const double* Xe = X + e * xs_e + size_t(x0 + a0) * n;
  const double* Ye = Y + e * ys_e + size_t(y0) * n;
  const int r0 = ch * rch, r1 = min(n, r0 + rch);
  double acc[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j) { acc[j][0] = 0.0; acc[j][1] = 0.0; }
  double px[LX], py[LY];
  auto fetch = [&](int rb) {
#pragma unroll
    for (int q = 0; q < LX; ++q) {
      const int idx = t + q * PEXP_THREADS, c = idx / 16, k = idx % 16, row = rb + k;
      px[q] = (a0 + c < nx && row < r1) ? __ldcg(Xe + size_t(c) * n + row) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < LY; ++q) {
      const int idx = t + q * PEXP_THREADS, c = idx / 16, k = idx % 16, row = rb + k;
      py[q] = (idx < 16 * NYT && c < ny && row < r1) ? __ldcg(Ye + size_t(c) * n + row) : 0.0;
    }
  };
  if (r0 < r1) fetch(r0);
  for (int rb = r0; rb < r1; rb += 16) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < LX; ++q) {
      const int idx = t + q * PEXP_THREADS;
      Xs[idx % 16][idx / 16] = px[q];
    }
#pragma unroll
    for (int q = 0; q < LY; ++q) {
      const int idx = t + q * PEXP_THREADS;
      if (idx < 16 * NYT) Ys[idx % 16][idx / 16] = py[q];
    }
    __syncthreads();
    if (rb + 16 < r1) fetch(rb + 16);
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      const double af = Xs[kq * 4 + fc][warp * 8 + fr];
#pragma unroll
      for (int j = 0; j < NJ; ++j) dmma884(acc[j][0], acc[j][1], af, Ys[kq * 4 + fc][j * 8 + fr]);
    }
  }
  double* P = part + (size_t(e) * nch + ch) * size_t(nx) * ny;
  const int a = a0 + warp * 8 + fr;
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int b = j * 8 + 2 * fc + h;
      if (a < nx && b < ny) P[a + size_t(b) * nx] = acc[j][h];
    }
}

// ---------------------------------------------------------------- host wrappers
// Tall path plan: Y sub-chunks of rsub rows (<= 48 KB of shared memory), CTA row range rch
// (multiple of rsub) chosen for ~6 waves over 148 SMs; partial count E*nch stays small.
void xty_tall_plan(int n, int E, int nx, int ny, int& rsub, int& rch, int& nch) {
  rsub = std::max(128, std::min(2048, (48 * 1024 / 8) / std::max(ny, 1)) / 128 * 128);
  if (long(cdiv(n, rsub)) * E < 148 * 6)  // few evaluations: smaller chunks for more CTAs
    rsub = std::max(128, std::min(rsub, int(long(n) * E / (148 * 6)) / 128 * 128));
  long want = std::max(1L, long(148 * 6) / std::max(E, 1));  // chunks per eval
  long per = std::max(1L, long(cdiv(n, rsub)) / want);        // sub-chunks per CTA
  rch = int(per * rsub);
  nch = cdiv(n, rch);
  (void)nx;
}

int xty_chunks(int n, int E) {
  // aim for >= ~4 waves of CTAs over 148 SMs, chunks of >= 512 rows
  int rch = 512;
  while (long(cdiv(n, rch)) * E > 148 * 8 && rch < n) rch *= 2;
  return rch;
}

void launch_xty(cudaStream_t st, int E, int n, const double* X, long long xs_e, int x0, int nx,
                const double* Y, long long ys_e, int y0, int ny, double* part, size_t part_cap,
                double* D, long long ds_e, int ldd, int row0, int col0, bool accumulate,
                const int* active, int* cnt) {
  if (E == 0 || nx == 0 || ny == 0) return;
  if (ny > 32 && ny <= 64 && stream_ok(n, 32) && stream_part_doubles(E, n, nx, 32) <= part_cap) {
    // wide right-hand blocks (the s = 64 source Grams of the SVD stage): two passes of the streaming
    // kernel over 32-column halves of Y (X is streamed twice; still ~3x faster than the register-tiled
    // square-Gram kernel on long columns)
    for (int h0 = 0; h0 < ny; h0 += 32) {
      const int nh = std::min(32, ny - h0);
      launch_sproj(st, E, n, X + size_t(x0) * n, xs_e, nx, Y + size_t(y0 + h0) * n, ys_e, nh, part, part_cap, D, ds_e,
                   ldd, row0, col0 + h0, accumulate, nullptr, 0, active);
    }
    return;
  }
  if (stream_ok(n, ny)) {  // TMA-fed DMMA streaming kernels (stream.cu)
    const bool gram = X == Y && xs_e == ys_e && x0 == y0 && nx == ny;
    const int pw = gram ? ny : nx;
    if (stream_part_doubles(E, n, pw, ny) <= part_cap) {
      if (gram)
        launch_sproj(st, E, n, X, xs_e, 0, Y + size_t(y0) * n, ys_e, ny, part, part_cap, nullptr, 0, 0, 0, 0, false, D,
                     ds_e, active, ldd, row0, col0);
      else
        launch_sproj(st, E, n, X + size_t(x0) * n, xs_e, nx, Y + size_t(y0) * n, ys_e, ny, part, part_cap, D, ds_e, ldd,
                     row0, col0, accumulate, nullptr, 0, active);
      return;
    }
  }
  RedArgs ra{D, ds_e, ldd, row0, col0, accumulate ? 1 : 0, cnt};
  if (ny > 8 && ny <= 32 && nx >= 32) {
    const int rch = xty_chunks(n, E * cdiv(nx, 64));
    const int nch = cdiv(n, rch);
    if (size_t(E) * nch * nx * ny > part_cap) fail(2, "xty partial buffer too small");
    const bool same = (X == Y && xs_e == ys_e && y0 >= x0 && y0 + ny <= x0 + nx);
    ProfScope ps(PC_XTY, st, eact(E, active) * n * 8.0 * (nx + (same ? 0 : ny)), 2.0 * eact(E, active) * double(n) * nx * ny);
    dim3 grid(nch, cdiv(nx, 64), E);
    if (ny <= 16)
      k_xty_mma<16><<<grid, PEXP_THREADS, 0, st>>>(n, rch, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active);
    else
      k_xty_mma<32><<<grid, PEXP_THREADS, 0, st>>>(n, rch, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active);
    count_launch();
    PEXP_LAUNCH_CHECK();
    dim3 g2(std::min(cdiv(nx * ny, PEXP_THREADS), 64), E);
    k_reduce<<<g2, PEXP_THREADS, 0, st>>>(nx, ny, nch, part, D, ds_e, ldd, row0, col0, accumulate ? 1 : 0, active);
    count_launch();
    PEXP_LAUNCH_CHECK();
    return;
  }
  if (ny <= 32) {
    int rsub, rch, nch;
    xty_tall_plan(n, E, nx, ny, rsub, rch, nch);
    if (size_t(E) * nch * nx * ny > part_cap) fail(2, "xty partial buffer too small");
    const bool same = (X == Y && xs_e == ys_e && y0 >= x0 && y0 + ny <= x0 + nx);
    ProfScope ps(PC_XTY, st, eact(E, active) * n * 8.0 * (nx + (same ? 0 : ny)), 2.0 * eact(E, active) * double(n) * nx * ny);
    size_t smem = (size_t(rsub) * ny + size_t(nx) * ny) * sizeof(double);
    if (smem > 200 * 1024) fail(1, "xty: nx*ny too large for the tall path");
    dim3 grid(nch, E);
    if (ny <= 4)
      k_xty_tall<4><<<grid, PEXP_THREADS, smem, st>>>(n, rch, rsub, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active, ra);
    else if (ny <= 8)
      k_xty_tall<8><<<grid, PEXP_THREADS, smem, st>>>(n, rch, rsub, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active, ra);
    else if (ny <= 16)
      k_xty_tall<16><<<grid, PEXP_THREADS, smem, st>>>(n, rch, rsub, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active, ra);
    else
      k_xty_tall<32><<<grid, PEXP_THREADS, smem, st>>>(n, rch, rsub, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active, ra);
    count_launch();
    PEXP_LAUNCH_CHECK();
    if (!cnt) {
      dim3 g2(std::min(cdiv(nx * ny, PEXP_THREADS), 64), E);
      k_reduce<<<g2, PEXP_THREADS, 0, st>>>(nx, ny, nch, part, D, ds_e, ldd, row0, col0, accumulate ? 1 : 0, active);
      count_launch();
      PEXP_LAUNCH_CHECK();
    }
    return;
  }
  int rch = xty_chunks(n, E);
  int nch = cdiv(n, rch);
  if (size_t(E) * nch * nx * ny > part_cap) fail(2, "xty partial buffer too small");
  int nxp = cdiv(nx, RA) * RA, nyp = cdiv(ny, RB) * RB;
  int ntiles = (nxp / RA) * (nyp / RB);
  size_t smem = size_t(TR) * (nxp + nyp) * sizeof(double);
  const bool same = (X == Y && xs_e == ys_e && y0 >= x0 && y0 + ny <= x0 + nx);
  ProfScope ps(PC_XTY, st, eact(E, active) * n * 8.0 * (nx + (same ? 0 : ny)), 2.0 * eact(E, active) * double(n) * nx * ny);
  dim3 grid(nch, E);
  if (nx > 32 && ny > 32 && nx <= 64 && ny <= 64) {
    k_xty_sq<<<grid, PEXP_THREADS, 0, st>>>(n, rch, X, xs_e, x0, nx, Y, ys_e, y0, ny, part);
  } else if (ntiles <= PEXP_THREADS) {
    k_xty_partial<1><<<grid, PEXP_THREADS, smem, st>>>(n, rch, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active);
  } else if (ntiles <= 2 * PEXP_THREADS) {
    k_xty_partial<2><<<grid, PEXP_THREADS, smem, st>>>(n, rch, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active);
  } else if (ntiles <= 4 * PEXP_THREADS) {
    k_xty_partial<4><<<grid, PEXP_THREADS, smem, st>>>(n, rch, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active);
  } else if (ntiles <= 8 * PEXP_THREADS) {
    k_xty_partial<8><<<grid, PEXP_THREADS, smem, st>>>(n, rch, X, xs_e, x0, nx, Y, ys_e, y0, ny, part, active);
  } else {
    fail(1, "xty: product too large (nx*ny > 32768)");
  }
  count_launch();
  PEXP_LAUNCH_CHECK();
  dim3 g2(std::min(cdiv(nx * ny, PEXP_THREADS), 64), E);
  k_reduce<<<g2, PEXP_THREADS, 0, st>>>(nx, ny, nch, part, D, ds_e, ldd, row0, col0, accumulate ? 1 : 0, active);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void launch_combine(cudaStream_t st, int E, int n, const double* X, long long xs_e, int x0, int nx,
                    const double* M, long long ms_e, int ldm, double* O, long long os_e, int o0,
                    int ny, double alpha, double beta, const int* active, const int* nxe) {
  if (E == 0 || ny == 0) return;
  if (stream_ok(n, std::min(ny, NB))) {  // TMA-fed DMMA streaming kernels (stream.cu)
    for (int b0 = 0; b0 < ny; b0 += NB) {
      const int nb = std::min(NB, ny - b0);
      if (nx == 0 && beta == 1.0) continue;
      if (ny > NB && O == X && o0 < x0 + nx && x0 < o0 + ny && xs_e == os_e)
        fail(1, "combine: in-place product with more than 32 output columns");
      launch_supdate(st, E, n, X + size_t(x0) * n, xs_e, nx, M + size_t(b0) * ldm, ms_e, ldm, O + size_t(o0 + b0) * n,
                     os_e, nb, alpha, beta, active, nxe);
    }
    return;
  }
  for (int b0 = 0; b0 < ny; b0 += NB) {
    int nb = std::min(NB, ny - b0);
    if (nx == 0) {
      if (beta == 1.0) continue;
    }
    if (ny > NB && O == X && o0 < x0 + nx && x0 < o0 + ny && xs_e == os_e)
      fail(1, "combine: in-place product with more than 32 output columns");
    const int nbt = nb <= 4 ? 4 : nb <= 8 ? 8 : nb <= 16 ? 16 : 32;
    size_t smem = size_t(std::max(nx, 1)) * nbt * sizeof(double);
    ProfScope ps(PC_COMBINE, st, eact(E, active) * n * 8.0 * (nx + nb * (beta != 0.0 ? 2 : 1)),
                 2.0 * eact(E, active) * double(n) * nx * nb);
    dim3 grid(cdiv(n, 2 * PEXP_THREADS), E);
    const double* Mb = M + size_t(b0) * ldm;
    if (nbt == 4)
      k_combine<4><<<grid, PEXP_THREADS, smem, st>>>(n, X, xs_e, x0, nx, Mb, ms_e, ldm, O, os_e, o0 + b0, nb, alpha, beta, active, nxe);
    else if (nbt == 8)
      k_combine<8><<<grid, PEXP_THREADS, smem, st>>>(n, X, xs_e, x0, nx, Mb, ms_e, ldm, O, os_e, o0 + b0, nb, alpha, beta, active, nxe);
    else if (nbt == 16)
      k_combine<16><<<grid, PEXP_THREADS, smem, st>>>(n, X, xs_e, x0, nx, Mb, ms_e, ldm, O, os_e, o0 + b0, nb, alpha, beta, active, nxe);
    else
      k_combine<32><<<grid, PEXP_THREADS, smem, st>>>(n, X, xs_e, x0, nx, Mb, ms_e, ldm, O, os_e, o0 + b0, nb, alpha, beta, active, nxe);
    count_launch();
    PEXP_LAUNCH_CHECK();
  }
}

void tsmm_init() {
  // allow > 48 KB dynamic shared memory
  cudaFuncSetAttribute(k_xty_partial<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_xty_partial<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_xty_partial<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_xty_partial<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_combine<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_combine<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_combine<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_combine<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_xty_tall<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_xty_tall<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_xty_tall<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_xty_tall<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace pexp
