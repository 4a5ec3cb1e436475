// common.cuh — shared device/host helpers of the pexp library (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>

#define PEXP_THREADS 256

namespace pexp {

// ---------------------------------------------------------------- error plumbing
struct Error {
  int code;
  std::string msg;
};

#define PEXP_CUDA_TRY(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      throw ::pexp::Error{3, std::string(#expr) + ": " + cudaGetErrorString(_e)};    \
  } while (0)

extern bool g_sync_debug;  // PEXP_SYNC=1: synchronise after every launch (fault localisation)
#define PEXP_LAUNCH_CHECK()                                                          \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e == cudaSuccess && ::pexp::g_sync_debug) _e = cudaDeviceSynchronize();     \
    if (_e != cudaSuccess)                                                           \
      throw ::pexp::Error{3, std::string("kernel launch (") + __FILE__ + ":" +        \
                                 std::to_string(__LINE__) + "): " + cudaGetErrorString(_e)}; \
  } while (0)

inline void fail(int code, const std::string& m) { throw Error{code, m}; }

// ---------------------------------------------------------------- launch counter
extern thread_local long g_launches;
inline void count_launch() { ++g_launches; }

// ---------------------------------------------------------------- live profiler
// Kernel classes; bytes/flops are ALGORITHMIC (what the method must move/compute for the
// launch's shapes), timed with CUDA events on the launch stream.
enum ProfCat { PC_SOLVE = 0, PC_XTY = 1, PC_COMBINE = 2, PC_SMALL = 3, PC_SVDSMALL = 4, PC_STENCIL = 5,
               PC_FACTOR = 6, PC_ARNOLDI = 7, PC_SCAN = 8, PC_SMALLHOM = 9, PC_SPROJ = 10,
               PC_SUPDATE = 11, PC_SCANOUT = 12, PC_NCAT = 13 };
struct ProfRec {
  cudaEvent_t a, b;
  int cat;
  double bytes, flops;
};
extern bool g_prof_on;
extern std::vector<ProfRec> g_prof;
struct ProfScope {
  bool on;
  ProfRec r;
  cudaStream_t st;
  ProfScope(int cat, cudaStream_t s, double bytes, double flops) : on(g_prof_on), st(s) {
    if (!on) return;
    r.cat = cat; r.bytes = bytes; r.flops = flops;
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, st);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(r.b, st);
    g_prof.push_back(r);
  }
};

// ---------------------------------------------------------------- workspace
// Bump allocator over caller-owned device memory.  With base == nullptr it only
// measures (used by pexp_workspace_bytes so size and layout can never disagree).
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    size_t bytes = ((count * sizeof(T)) + 255) & ~size_t(255);
    size_t o = off;
    off += bytes;
    if (base == nullptr) return nullptr;
    if (off > cap) fail(2, "workspace too small (pexp_workspace_bytes underestimated?)");
    return reinterpret_cast<T*>(base + o);
  }
};

inline int cdiv(long a, long b) { return int((a + b - 1) / b); }

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `red` must hold >= 32 doubles; result broadcast to all threads.
__device__ __forceinline__ double block_sum(double v, double* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (w == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ double block_max(double v, double* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : -1.0e308;
  if (w == 0) t = warp_max(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

// atomic max for non-negative doubles (bit patterns of non-negative IEEE doubles are
// ordered like unsigned integers).
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

}  // namespace pexp
