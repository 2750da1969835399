// Shared helpers for the sm_100a TT-IGA kernels.
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>

namespace cg = cooperative_groups;

#define TTB_API extern "C" __attribute__((visibility("default")))
#include <stdio.h>
#include <stdlib.h>
// TTB_DEBUG_SYNC=1: synchronize after instrumented launches and report the first failing step
inline bool ttb_debug_sync() {
  static int v = -1;
  if (v < 0) v = getenv("TTB_DEBUG_SYNC") ? 1 : 0;
  return v == 1;
}
#define TTB_DBG(stream, what)                                                               \
  do {                                                                                     \
    if (ttb_debug_sync()) {                                                                \
      cudaError_t e_ = cudaStreamSynchronize(stream);                                      \
      if (e_ != cudaSuccess) fprintf(stderr, "ttb debug: %s failed: %d (%s:%d)\n", what, (int)e_, __FILE__, __LINE__); \
    }                                                                                      \
  } while (0)

// error codes returned through the C ABI (0 = ok, >0 = CUDA error, <0 = argument/numerical)
enum {
  TTB_OK = 0,
  TTB_EARG = -1,
  TTB_ENOTPD = -2,     // Cholesky hit a non-positive pivot
  TTB_ESINGULAR = -3,  // LU / maxvol hit a zero pivot
  TTB_ENOCONV = -4,
};

static inline int ttb_last_error() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

// host-side count of kernel launches issued by this library (bench.py's gpu_launches evidence)
extern long long g_ttb_launches;
static inline void ttb_count() { __atomic_add_fetch(&g_ttb_launches, 1LL, __ATOMIC_RELAXED); }

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device (grid sizes of grid-stride and persistent kernels; 148 on B200)
static inline int ttb_num_sms() {
  static int n = 0;
  if (!n) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n <= 0) n = 148;
  }
  return n;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp all-reduce of 16 values: reduce-scatter over lane bits 4..1 (lane l ends with the sum of
// index l >> 1), a final exchange over bit 0, then an all-gather: 64 shuffles instead of 160.
__device__ __forceinline__ void warp_allreduce16(double (&z)[16], int lane) {
  double v8[8], v4[4], v2[2];
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double send = hi ? z[k] : z[k + 8];
      const double keep = hi ? z[k + 8] : z[k];
      v8[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double send = hi ? v8[k] : v8[k + 4];
      const double keep = hi ? v8[k + 4] : v8[k];
      v4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double send = hi ? v4[k] : v4[k + 2];
      const double keep = hi ? v4[k + 2] : v4[k];
      v2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
  }
  double v;
  {
    const bool hi = lane & 2;
    const double send = hi ? v2[0] : v2[1];
    const double keep = hi ? v2[1] : v2[0];
    v = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  v += __shfl_xor_sync(0xffffffffu, v, 1);  // lane l: full sum of index l >> 1
#pragma unroll
  for (int c = 0; c < 16; ++c) z[c] = __shfl_sync(0xffffffffu, v, 2 * c);
}

// block-wide sum; result valid in every thread. smem must hold >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? smem[threadIdx.x] : 0.0;
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) smem[0] = t;
  __syncthreads();
  double r = smem[0];
  __syncthreads();
  return r;
}

// argmax of |value| with lowest-index tie-break (numpy argmax semantics).
struct AbsMax {
  double v;
  long long i;
};

__device__ __forceinline__ AbsMax absmax_merge(AbsMax a, AbsMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ __forceinline__ AbsMax warp_absmax(AbsMax a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    AbsMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = absmax_merge(a, b);
  }
  return a;
}

__device__ __forceinline__ AbsMax block_absmax(AbsMax a, double* sv, long long* si) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  a = warp_absmax(a);
  __syncthreads();
  if (lane == 0) { sv[wid] = a.v; si[wid] = a.i; }
  __syncthreads();
  if (wid == 0) {
    AbsMax b;
    b.v = lane < nw ? sv[lane] : -1.0;
    b.i = lane < nw ? si[lane] : (1LL << 62);
    b = warp_absmax(b);
    if (lane == 0) { sv[0] = b.v; si[0] = b.i; }
  }
  __syncthreads();
  AbsMax r;
  r.v = sv[0];
  r.i = si[0];
  __syncthreads();
  return r;
}

static inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }
