// Shared helpers for the sm_100a TT-IGA kernels.
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>

namespace cg = cooperative_groups;

#define TTB_API extern "C" __attribute__((visibility("default")))

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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
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
