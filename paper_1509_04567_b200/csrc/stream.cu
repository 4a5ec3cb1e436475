// stream.cu — the streaming route's tall-skinny products (subsystem 2, block classical
// Gram-Schmidt with reorthogonalisation, PAPER.md:171-176 Eq.(blockKrylovSubspace)) for long
// columns (C5: n = 65536), where the fused cluster step's block rows do not fit on chip:
//
//   k_sproj   : D = X^T Y  and  G = Y^T Y   (X = the basis V[:, 0:nx], Y = the new block, ny <= 32)
//   k_supdate : Y = beta Y + alpha X M       (M: nx x ny, e.g. W -= V H)
//
// Both are persistent, warp-specialised kernels: one producer warp streams the CTA's row chunk of
// X through a ring of shared-memory stages with 1D bulk TMA copies (cp.async.bulk, completion on
// mbarriers: UBLKCP in SASS), eight consumer warps run the contraction on the fp64 tensor cores
// (DMMA m8n8k4).  A stage holds 8 columns of X for R = 512 rows (each column one 4 KB bulk copy,
// column stride padded by 32 B so a fragment load is exactly two shared-memory wavefronts).
//
// k_sproj (ny <= 8): consumer warp w owns rows [64w, 64w + 64) of the chunk and keeps its Y rows as DMMA B
// fragments in registers for the whole item; per stage it accumulates the 8 x ny tile of X^T Y over
// its rows, the 8 warps' tiles are summed through shared memory in warp order and written as the
// chunk's partial; G = Y^T Y uses the same registers as A and B operands.  k_sproj2 (ny > 8, see there):
// warps own (column tile, row quarter) pairs and reduce behind per-tile named barriers, which keeps the
// DMMA pipe busy at the wide blocks where it is the limiter.  Partials are summed in chunk order by
// k_sred (deterministic, parallel over outputs).
// k_supdate: consumer warp w owns the same 64 rows; its D fragments (64 rows x ny) stay in
// registers across all stages (the sum over X's columns is the DMMA k-dimension), B fragments are
// the matching 8 rows of M per stage (L1/L2 resident), the epilogue writes beta Y + alpha acc.
//
// Requirements (checked by stream_ok): n even (16-byte aligned column starts for the bulk copies),
// ny <= 32.  Algorithmic bytes: X read once per launch (8 n nx), Y read once (and written once by
// k_supdate); DMMA flops 2 n nx ny (+ 2 n ny^2 for G).
#include "common.cuh"
#include "kernels.cuh"

namespace pexp {

namespace {

constexpr int SR = 512;                 // rows per work item (chunk)
constexpr int SCOLS = 8;                // X columns per stage
constexpr int SNW = 8;                  // consumer warps
constexpr int STHREADS = (SNW + 1) * 32;
constexpr int SNST = 4;                 // ring stages
constexpr int SCOL_STRIDE = SR + 4;     // doubles per staged column (32 B pad)
constexpr int SSTAGE = SCOLS * SCOL_STRIDE;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(SNW * 32) : "memory"); }

struct Item {
  int e, c;  // evaluation, row chunk
};

// Work items (e, c) with active[e] != 0, enumerated identically by producer and consumers.
__device__ __forceinline__ bool next_item(int& it, int nitems, int nch, const int* active, Item& w) {
  while (it < nitems) {
    const int e = it / nch, c = it % nch;
    if (!active || active[e]) {
      w.e = e;
      w.c = c;
      return true;
    }
    it += gridDim.x;
  }
  return false;
}

// One streamed segment of columns of a work item: columns [0, ncols) of P (per-eval stride s_e),
// rows [c*SR, c*SR + rows); ncols_e (nullable) caps the count per evaluation.
struct Seg {
  const double* P;
  long long s_e;
  int ncols;
  const int* ncols_e;
  __device__ int count(int e) const { return P ? (ncols_e ? min(ncols, ncols_e[e]) : ncols) : 0; }
};

// Producer (one lane): for every item, segment a then segment b, 8 columns per stage, each column
// one bulk copy of the item's rows into the ring.
__device__ void produce(int n, int nitems, int nch, const int* active, Seg sa, Seg sb, double* ring,
                        unsigned long long* full, unsigned long long* empty) {
  if ((threadIdx.x & 31) != 0) return;
  int slot = 0;
  unsigned ph = 0;
  Item w;
  for (int it = blockIdx.x; next_item(it, nitems, nch, active, w); it += gridDim.x) {
    const int r0 = w.c * SR, rows = min(SR, n - r0);
    const unsigned bytes = unsigned(rows) * 8u;
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      const Seg& sg = q == 0 ? sa : sb;
      const int nx = sg.count(w.e);
      const double* Xe = sg.P + w.e * sg.s_e + r0;
      for (int g = 0; g < nx; g += SCOLS) {
        const int nc = min(SCOLS, nx - g);
        mbar_wait(&empty[slot], ph ^ 1u);
        mbar_expect_tx(&full[slot], bytes * nc);
        double* st = ring + size_t(slot) * SSTAGE;
        for (int k = 0; k < nc; ++k) bulk_g2s(st + k * SCOL_STRIDE, Xe + size_t(g + k) * n, bytes, &full[slot]);
        if (++slot == SNST) { slot = 0; ph ^= 1u; }
      }
    }
  }
}

// Consumer-side ring position.
struct RingPos {
  int slot = 0;
  unsigned ph = 0;
  __device__ void advance() {
    if (++slot == SNST) { slot = 0; ph ^= 1u; }
  }
};

// Shared-memory ring setup: zero the stages and init the barriers.  Called by all threads.
// Rows of a short last chunk beyond n are never copied: the stage keeps zeros or finite basis
// values of an earlier item there, which meet zero Y fragments (k_sproj) or feed output rows
// that are not stored (k_supdate).
__device__ void ring_setup(double* ring, unsigned long long* full, unsigned long long* empty) {
  for (int i = threadIdx.x; i < SNST * SSTAGE; i += blockDim.x) ring[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SNST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SNW);
    }
  }
  fence_proxy_async();
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
}

}  // namespace

// ---------------------------------------------------------------- D = X^T Y, G = Y^T Y partials
// part[(e * nch + c) * (nx + ny) * ny + a + b * (nx + ny)]: a < nx -> (X^T Y)[a][b], a >= nx -> (Y^T Y)[a - nx][b]
// Ring order per item: the ceil(ny/8) stages of Y (loaded into B fragments), then the X stages.
template <int MB>
__global__ void __launch_bounds__(STHREADS, 1)
k_sproj(int E, int n, int nch, const double* X, long long xs_e, int nx, const double* Y, long long ys_e, int ny,
        int gram, double* part, const int* active) {
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;
  double* red = ring + SNST * SSTAGE;  // [2][SNW][8][MB + 8] warp tiles (double-buffered over the stages)
  int rbuf = 0;
  __shared__ __align__(8) unsigned long long full[SNST], empty[SNST];
  ring_setup(ring, full, empty);
  const int nitems = E * nch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == SNW) {
    produce(n, nitems, nch, active, Seg{Y, ys_e, ny, nullptr}, Seg{X, xs_e, nx, nullptr}, ring, full, empty);
    return;
  }
  constexpr int NJ = MB / 8;
  constexpr int MBP = MB + 8;  // tile row stride: consecutive rows 64 B apart modulo 128 B (conflict-free)
  const int njt = (ny + 7) >> 3;
  const int pw = nx + (gram ? ny : 0);
  RingPos rp;
  Item w;
  for (int it = blockIdx.x; next_item(it, nitems, nch, active, w); it += gridDim.x) {
    const int r0 = w.c * SR, rows = min(SR, n - r0);
    // B fragments from the Y stages: Y[row 64w + 4q + (lane&3)][col 8j + (lane>>2)]
    double bf[16][NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if (j < njt) {
        mbar_wait(&full[rp.slot], rp.ph);
        const double* st = ring + size_t(rp.slot) * SSTAGE + (lane >> 2) * SCOL_STRIDE + 64 * warp + (lane & 3);
        const bool colok = 8 * j + (lane >> 2) < ny;
#pragma unroll
        for (int q = 0; q < 16; ++q) bf[q][j] = (colok && 64 * warp + 4 * q + (lane & 3) < rows) ? st[4 * q] : 0.0;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rp.slot]);
        rp.advance();
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) bf[q][j] = 0.0;
      }
    }
    double* P = part + size_t(w.e * nch + w.c) * pw * ny;
    const bool rows_here = 64 * warp < rows;
    for (int g = 0; g < nx; g += SCOLS) {
      double acc[NJ][2];
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = 0.0;
      mbar_wait(&full[rp.slot], rp.ph);
      const double* st = ring + size_t(rp.slot) * SSTAGE + (lane >> 2) * SCOL_STRIDE + 64 * warp + (lane & 3);
      if (rows_here) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const double a = st[4 * q];
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (j < njt) dmma(acc[j][0], acc[j][1], a, bf[q][j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rp.slot]);
      rp.advance();
      // warp tiles -> shared (D[i = lane>>2][jcol = 8j + 2(lane&3) + h]); sum in warp order.  The tile
      // buffer is double-buffered over the stages, so ONE consumer barrier per stage suffices (the
      // barrier of stage g+1 orders the reads of buffer b before the writes of stage g+2 into it)
      double* rb = red + rbuf * (SNW * 8 * MBP);
      rbuf ^= 1;
      double* rw = rb + warp * (8 * MBP);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        rw[(lane >> 2) * MBP + 8 * j + 2 * (lane & 3)] = acc[j][0];
        rw[(lane >> 2) * MBP + 8 * j + 2 * (lane & 3) + 1] = acc[j][1];
      }
      consumer_sync();
      const int nc = min(SCOLS, nx - g);
      for (int idx = threadIdx.x; idx < nc * ny; idx += SNW * 32) {
        const int b = idx % ny, i = idx / ny;   // consecutive threads -> consecutive tile columns
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < SNW; ++q) s += rb[q * (8 * MBP) + i * MBP + b];
        P[(g + i) + size_t(b) * pw] = s;
      }
    }
    consumer_sync();  // the Gram tiles below reuse buffer 0
    if (gram) {  // G = Y^T Y over the chunk: A fragment of tile i = bf[q][i] (same layout)
#pragma unroll
      for (int i = 0; i < NJ; ++i) {
        if (i >= njt) break;
        double acc[NJ][2];
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (j < njt) dmma(acc[j][0], acc[j][1], bf[q][i], bf[q][j]);
        double* rw = red + warp * (8 * MBP);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          rw[(lane >> 2) * MBP + 8 * j + 2 * (lane & 3)] = acc[j][0];
          rw[(lane >> 2) * MBP + 8 * j + 2 * (lane & 3) + 1] = acc[j][1];
        }
        consumer_sync();
        const int nc = min(8, ny - 8 * i);
        for (int idx = threadIdx.x; idx < nc * ny; idx += SNW * 32) {
          const int b = idx % ny, ii = idx / ny;
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < SNW; ++q) s += red[q * (8 * MBP) + ii * MBP + b];
          P[nx + 8 * i + ii + size_t(b) * pw] = s;
        }
        consumer_sync();
      }
    }
  }
}

// ---------------------------------------------------------------- wide blocks (ny > 8): k_sproj2
// Same product and partial layout as k_sproj, with the work split so that the fp64 tensor pipe never
// waits for a CTA-wide reduction: 4 NJ consumer warps, warp (tj, q) = (w / 4, w % 4) owns the 8-column
// tile tj of Y and the row quarter q (128 rows) of the chunk (the four quarters of a tile sit on the four
// SM sub-partitions, every sub-partition hosts one warp per tile).  Its Y rows are DMMA B fragments in 64
// registers; per X stage it issues 32 DMMAs and the four quarter tiles are summed through shared memory
// behind a 128-thread NAMED barrier of that tile group only -- the other tile groups keep the tensor
// pipe busy meanwhile.  G = Y^T Y uses the Y stages themselves as A operands (they stay in the ring
// until every tile pair is done), so a warp never needs another tile's fragments.
constexpr int SNST2 = 6;  // ring stages (the Y stages of an item, up to 4, stay resident during the Gram)
template <int NJ>
__global__ void __launch_bounds__((4 * NJ + 1) * 32, 1)
k_sproj2(int E, int n, int nch, const double* X, long long xs_e, int nx, const double* Y, long long ys_e, int ny,
         int gram, double* part, const int* active) {
  constexpr int NCW = 4 * NJ;
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;
  double* red = ring + SNST2 * SSTAGE;  // [2][NJ][4][64] quarter tiles (double-buffered over the stages)
  __shared__ __align__(8) unsigned long long full[SNST2], empty[SNST2];
  for (int i = threadIdx.x; i < SNST2 * SSTAGE; i += blockDim.x) ring[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < SNST2; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], NCW);
    }
  }
  fence_proxy_async();
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  const int nitems = E * nch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int njt = (ny + 7) >> 3;
  if (warp == NCW) {  // producer: the Y stages, then the X stages of every item
    if (lane != 0) return;
    int slot = 0;
    unsigned ph = 0;
    Item w;
    for (int it = blockIdx.x; next_item(it, nitems, nch, active, w); it += gridDim.x) {
      const int r0 = w.c * SR, rows = min(SR, n - r0);
      const unsigned bytes = unsigned(rows) * 8u;
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const double* Pe = q == 0 ? Y + w.e * ys_e + r0 : X + w.e * xs_e + r0;
        const int ncol = q == 0 ? ny : nx;
        for (int g = 0; g < ncol; g += SCOLS) {
          const int nc = min(SCOLS, ncol - g);
          mbar_wait(&empty[slot], ph ^ 1u);
          mbar_expect_tx(&full[slot], bytes * nc);
          double* st = ring + size_t(slot) * SSTAGE;
          for (int k = 0; k < nc; ++k) bulk_g2s(st + k * SCOL_STRIDE, Pe + size_t(g + k) * n, bytes, &full[slot]);
          if (++slot == SNST2) { slot = 0; ph ^= 1u; }
        }
      }
    }
    return;
  }
  const int tj = warp >> 2, q4 = warp & 3;
  const bool tile_on = tj < njt;
  const int pw = nx + (gram ? ny : 0);
  int slot = 0, rbuf = 0;
  unsigned ph = 0;
  auto advance = [&]() {
    if (++slot == SNST2) { slot = 0; ph ^= 1u; }
  };
  // quarter tiles of one 8 x 8 output block -> partial rows [orow, orow + nrow) x columns of tile tj
  auto reduce_store = [&](double a0, double a1, double* P, int orow, int nrow) {
    double* rb = red + size_t(rbuf) * (NJ * 4 * 64) + tj * (4 * 64);
    rbuf ^= 1;
    rb[q4 * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = a0;
    rb[q4 * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = a1;
    asm volatile("bar.sync %0, 128;\n" ::"r"(1 + tj) : "memory");
    const int t = q4 * 32 + lane;  // 0..127 within the tile group; the first 64 threads own one output each
    if (t < 64) {
      const int m = t & 7, nn = t >> 3;  // consecutive threads -> consecutive partial rows (coalesced)
      const double s4 = (rb[m * 8 + nn] + rb[64 + m * 8 + nn]) + (rb[128 + m * 8 + nn] + rb[192 + m * 8 + nn]);
      if (m < nrow && 8 * tj + nn < ny) P[(orow + m) + size_t(8 * tj + nn) * pw] = s4;
    }
  };
  Item w;
  for (int it = blockIdx.x; next_item(it, nitems, nch, active, w); it += gridDim.x) {
    const int r0 = w.c * SR, rows = min(SR, n - r0);
    double* P = part + size_t(w.e * nch + w.c) * pw * ny;
    // ---- Y stages: B fragments of the warp's tile; the stages stay in the ring for the Gram
    const int yslot0 = slot;
    const unsigned yph0 = ph;
    double bf[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) bf[k] = 0.0;
    for (int j = 0; j < njt; ++j) {
      mbar_wait(&full[slot], ph);
      if (j == tj) {
        const double* st = ring + size_t(slot) * SSTAGE + (lane >> 2) * SCOL_STRIDE + 128 * q4 + (lane & 3);
        const bool colok = 8 * j + (lane >> 2) < ny;
#pragma unroll
        for (int k = 0; k < 32; ++k) bf[k] = (colok && 128 * q4 + 4 * k + (lane & 3) < rows) ? st[4 * k] : 0.0;
      }
      advance();
    }
    if (gram) {  // G[8 i + m][8 tj + nn] = sum_rows Y_i[row][m] Y_tj[row][nn]: A from the resident Y stage i
      int gs = yslot0;
      for (int i = 0; i < njt; ++i) {
        double a0 = 0.0, a1 = 0.0;
        if (tile_on) {
          const double* st = ring + size_t(gs) * SSTAGE + (lane >> 2) * SCOL_STRIDE + 128 * q4 + (lane & 3);
          const bool colok = 8 * i + (lane >> 2) < ny;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const double a = (colok && 128 * q4 + 4 * k + (lane & 3) < rows) ? st[4 * k] : 0.0;
            dmma(a0, a1, a, bf[k]);
          }
          reduce_store(a0, a1, P, nx + 8 * i, min(8, ny - 8 * i));
        }
        if (++gs == SNST2) gs = 0;
      }
    }
    {  // release the Y stages
      int rs = yslot0;
      __syncwarp();
      for (int j = 0; j < njt; ++j) {
        if (lane == 0) mbar_arrive(&empty[rs]);
        if (++rs == SNST2) rs = 0;
      }
      (void)yph0;
    }
    // ---- X stages
    for (int g = 0; g < nx; g += SCOLS) {
      double a0 = 0.0, a1 = 0.0;
      mbar_wait(&full[slot], ph);
      if (tile_on && 128 * q4 < rows) {
        const double* st = ring + size_t(slot) * SSTAGE + (lane >> 2) * SCOL_STRIDE + 128 * q4 + (lane & 3);
#pragma unroll
        for (int k = 0; k < 32; ++k) dmma(a0, a1, st[4 * k], bf[k]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      advance();
      if (tile_on) reduce_store(a0, a1, P, g, min(SCOLS, nx - g));
    }
  }
}

// Output descriptor of a reduced block: element (a, b) -> p[e * s_e + (row0 + a) + (col0 + b) * ld].
struct OutDesc {
  double* p;
  long long s_e;
  int ld, row0, col0, accumulate;
};

// Sum the chunk partials in chunk order: rows a < nx -> D, rows a >= nx -> G (row a - nx).
__global__ void k_sred(int nx, int ny, int pw, int nch, const double* part, OutDesc D, OutDesc G, const int* active) {
  const int e = blockIdx.y;
  if (active && !active[e]) return;
  const size_t sz = size_t(pw) * ny;
  const double* pe = part + size_t(e) * nch * sz;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < pw * ny; idx += gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    int c = 0;
    for (; c + 1 < nch; c += 2) {
      s0 += __ldcg(pe + size_t(c) * sz + idx);
      s1 += __ldcg(pe + size_t(c + 1) * sz + idx);
    }
    if (c < nch) s0 += __ldcg(pe + size_t(c) * sz + idx);
    const double s = s0 + s1;
    int a = idx % pw;
    const int b = idx / pw;
    const OutDesc& o = a < nx ? D : G;
    if (a >= nx) a -= nx;
    double* d = o.p + e * o.s_e + (o.row0 + a) + size_t(o.col0 + b) * o.ld;
    *d = o.accumulate ? *d + s : s;
  }
}

// ---------------------------------------------------------------- Y = beta Y + alpha X M
// Ring order per item: the X stages, then (beta != 0) the ceil(ny/8) stages of Y's old values.
template <int MB>
__global__ void __launch_bounds__(STHREADS, 1)
k_supdate(int E, int n, int nch, const double* X, long long xs_e, int nx0, const double* M, long long ms_e, int ldm,
          double* Y, long long ys_e, int ny, double alpha, double beta, const int* active, const int* nxe) {
  extern __shared__ __align__(16) double sm[];
  double* ring = sm;
  __shared__ __align__(8) unsigned long long full[SNST], empty[SNST];
  ring_setup(ring, full, empty);
  const int nitems = E * nch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == SNW) {
    produce(n, nitems, nch, active, Seg{X, xs_e, nx0, nxe}, Seg{beta != 0.0 ? Y : nullptr, ys_e, ny, nullptr}, ring,
            full, empty);
    return;
  }
  constexpr int NJ = MB / 8;
  const int njt = (ny + 7) >> 3;
  RingPos rp;
  Item w;
  for (int it = blockIdx.x; next_item(it, nitems, nch, active, w); it += gridDim.x) {
    const int r0 = w.c * SR, rows = min(SR, n - r0);
    const double* Me = M + w.e * ms_e;
    const int nx = nxe ? min(nx0, nxe[w.e]) : nx0;
    double acc[8][NJ][2];
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[t][j][0] = acc[t][j][1] = 0.0;
    const bool rows_here = 64 * warp < rows;
    // B fragments M[g + 4kq + (lane&3)][8j + (lane>>2)] (zero beyond nx / ny), one stage ahead
    double bm[2][NJ], bn[2][NJ];
    auto load_bm = [&](int g, double (&d)[2][NJ]) {
#pragma unroll
      for (int kq = 0; kq < 2; ++kq) {
        const int a = g + 4 * kq + (lane & 3);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int b = 8 * j + (lane >> 2);
          d[kq][j] = (a < nx && b < ny) ? __ldg(Me + a + size_t(b) * ldm) : 0.0;
        }
      }
    };
    constexpr bool PREF = NJ <= 2;  // prefetching M one stage ahead pays only below MB = 32 (measured: 2.58 vs 2.70 s on C5)
    if (PREF) load_bm(0, bm);
    for (int g = 0; g < nx; g += SCOLS) {
      if (PREF)
        load_bm(g + SCOLS, bn);
      else
        load_bm(g, bm);
      mbar_wait(&full[rp.slot], rp.ph);
      // A fragment: X[col 4kq + (lane&3)][row 64w + 8t + (lane>>2)]
      const double* st = ring + size_t(rp.slot) * SSTAGE + (lane & 3) * SCOL_STRIDE + 64 * warp + (lane >> 2);
      if (rows_here) {
#pragma unroll
        for (int kq = 0; kq < 2; ++kq)
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const double a = st[kq * 4 * SCOL_STRIDE + 8 * t];
#pragma unroll
            for (int j = 0; j < NJ; ++j)
              if (j < njt) dmma(acc[t][j][0], acc[t][j][1], a, bm[kq][j]);
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rp.slot]);
      rp.advance();
      if (PREF)
#pragma unroll
        for (int kq = 0; kq < 2; ++kq)
#pragma unroll
          for (int j = 0; j < NJ; ++j) bm[kq][j] = bn[kq][j];
    }
    // epilogue: D[row 8t + (lane>>2)][col 8j + 2(lane&3) + h]; old Y values from the Y stages
    double* Ye = Y + w.e * ys_e + r0;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      if (j >= njt) break;
      const double* sy = nullptr;
      if (beta != 0.0) {
        mbar_wait(&full[rp.slot], rp.ph);
        sy = ring + size_t(rp.slot) * SSTAGE + 64 * warp + (lane >> 2);
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int r = 64 * warp + 8 * t + (lane >> 2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cb = 2 * (lane & 3) + h, b = 8 * j + cb;
          if (b < ny && r < rows) {
            double v = alpha * acc[t][j][h];
            if (beta != 0.0) v = fma(beta, sy[cb * SCOL_STRIDE + 8 * t], v);
            Ye[size_t(b) * n + r] = v;
          }
        }
      }
      if (beta != 0.0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rp.slot]);
        rp.advance();
      }
    }
  }
}

// ---------------------------------------------------------------- host side
bool stream_ok(int n, int ny) { return (n % 2) == 0 && ny >= 1 && ny <= 32 && n >= SR; }

static int stream_grid(int items) { return std::max(1, std::min(items, 148)); }

static size_t sproj_smem(int MB) { return sizeof(double) * (size_t(SNST) * SSTAGE + 2 * size_t(SNW) * 8 * (MB + 8)); }
static size_t supdate_smem() { return sizeof(double) * size_t(SNST) * SSTAGE; }
static size_t sproj2_smem(int NJ) { return sizeof(double) * (size_t(SNST2) * SSTAGE + 2 * size_t(NJ) * 4 * 64); }

// partial doubles of E evaluations when pw rows (nx, plus ny if the Gram is fused) x ny are reduced
size_t stream_part_doubles(int E, int n, int pw, int ny) { return size_t(E) * cdiv(n, SR) * size_t(pw) * ny; }

void launch_sproj(cudaStream_t st, int E, int n, const double* X, long long xs_e, int nx, const double* Y,
                  long long ys_e, int ny, double* part, size_t part_cap, double* D, long long ds_e, int ldd, int row0,
                  int col0, bool accumulate, double* G, long long gs_e, const int* active, int gld, int grow0,
                  int gcol0) {
  if (gld <= 0) gld = ny;
  if (E == 0 || ny == 0 || (nx == 0 && !G)) return;
  if (!stream_ok(n, ny)) fail(1, "streaming projection: unsupported shape");
  const int nch = cdiv(n, SR);
  const int pw = nx + (G ? ny : 0);
  if (size_t(E) * nch * pw * ny > part_cap) fail(2, "streaming projection: partial buffer too small");
  const double ea = eact(E, active);
  {
    ProfScope ps(PC_SPROJ, st, ea * n * 8.0 * (nx + ny), 2.0 * ea * double(n) * ny * (nx + (G ? ny : 0)));
    const int gx = stream_grid(E * nch);
    const int MB = ny <= 8 ? 8 : ny <= 16 ? 16 : 32;
    const int gram = G ? 1 : 0;
    if (MB == 8)
      k_sproj<8><<<gx, STHREADS, sproj_smem(8), st>>>(E, n, nch, X, xs_e, nx, Y, ys_e, ny, gram, part, active);
    else if (ny <= 16)
      k_sproj2<2><<<gx, 9 * 32, sproj2_smem(2), st>>>(E, n, nch, X, xs_e, nx, Y, ys_e, ny, gram, part, active);
    else if (ny <= 24)
      k_sproj2<3><<<gx, 13 * 32, sproj2_smem(3), st>>>(E, n, nch, X, xs_e, nx, Y, ys_e, ny, gram, part, active);
    else
      k_sproj2<4><<<gx, 17 * 32, sproj2_smem(4), st>>>(E, n, nch, X, xs_e, nx, Y, ys_e, ny, gram, part, active);
    count_launch();
    PEXP_LAUNCH_CHECK();
    dim3 g2(std::min(cdiv(pw * ny, 256), 16), E);
    const OutDesc od{D, ds_e, ldd, row0, col0, accumulate ? 1 : 0};
    const OutDesc og{G, gs_e, gld, grow0, gcol0, (nx == 0 && accumulate) ? 1 : 0};
    k_sred<<<g2, 256, 0, st>>>(nx, ny, pw, nch, part, od, og, active);
    count_launch();
    PEXP_LAUNCH_CHECK();
  }
}

void launch_supdate(cudaStream_t st, int E, int n, const double* X, long long xs_e, int nx, const double* M,
                    long long ms_e, int ldm, double* Y, long long ys_e, int ny, double alpha, double beta,
                    const int* active, const int* nxe) {
  if (E == 0 || ny == 0) return;
  if (!stream_ok(n, ny)) fail(1, "streaming update: unsupported shape");
  const int nch = cdiv(n, SR);
  const double ea = eact(E, active);
  ProfScope ps(PC_SUPDATE, st, ea * n * 8.0 * (nx + ny * (beta != 0.0 ? 2 : 1)), 2.0 * ea * double(n) * nx * ny);
  const int gx = stream_grid(E * nch);
  const int MB = ny <= 8 ? 8 : ny <= 16 ? 16 : 32;
  if (MB == 8)
    k_supdate<8><<<gx, STHREADS, supdate_smem(), st>>>(E, n, nch, X, xs_e, nx, M, ms_e, ldm, Y, ys_e, ny, alpha, beta,
                                                       active, nxe);
  else if (MB == 16)
    k_supdate<16><<<gx, STHREADS, supdate_smem(), st>>>(E, n, nch, X, xs_e, nx, M, ms_e, ldm, Y, ys_e, ny, alpha,
                                                        beta, active, nxe);
  else
    k_supdate<32><<<gx, STHREADS, supdate_smem(), st>>>(E, n, nch, X, xs_e, nx, M, ms_e, ldm, Y, ys_e, ny, alpha,
                                                        beta, active, nxe);
  count_launch();
  PEXP_LAUNCH_CHECK();
}

void stream_init() {
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_sproj<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sproj_smem(8)));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_sproj<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sproj_smem(16)));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_sproj<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sproj_smem(32)));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_sproj2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sproj2_smem(2)));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_sproj2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sproj2_smem(3)));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_sproj2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sproj2_smem(4)));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_supdate<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)supdate_smem()));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_supdate<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)supdate_smem()));
  PEXP_CUDA_TRY(cudaFuncSetAttribute(k_supdate<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)supdate_smem()));
}

}  // namespace pexp
