// INT8 tensor-core GEMM on the 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM
// accumulators): C (int32, M x N row-major) = A (int8, M x K row-major) * B (int8, N x K row-major)^T.
// Building block for FP64 emulation by the Ozaki scheme (exact int32 accumulation of int8 slices).
//
// Operand tiles of 128 (or 256) rows x 128 bytes of K live in shared memory in the 128-byte-swizzled
// K-major layout (row r, 16-byte chunk c at r * 128 + ((c ^ (r & 7)) * 16)) that the SM100 matrix
// descriptors (version 1, SBO 1024) describe; one thread issues 4 MMAs (K = 32 each) per stage and
// commits them to that stage's mbarrier, which gates the reuse of the stage. Default: TMA loads
// (cp.async.bulk.tensor, hardware swizzle) into a 4-stage ring, 128 x 256 tiles (2.25 POPS on
// 8192^3); fallback / TTB_I8GEMM=s: synchronous loads by all threads, 128 x 128 tiles, 2 stages.
#include "common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>

namespace {

constexpr int I8_BM = 128, I8_BN = 128, I8_BK = 128, I8_T = 128, I8_ST = 2;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, 128-byte swizzle, 8-row core groups 1024 bytes apart (SM100 descriptor version 1)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::i8 instruction descriptor: D s32, A/B signed int8, both K-major, N = 128, M = 128
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(I8_BN >> 3) << 17) |
                              ((uint32_t)(I8_BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescI8), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}\n" ::"r"(mbar),
      "r"(phase));
}

__global__ void __launch_bounds__(I8_T, 1) i8gemm_kernel(int M, int N, int K, const int8_t* __restrict__ A,
                                                       const int8_t* __restrict__ B, int* __restrict__ C) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t mbar[I8_ST];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * I8_BM, n0 = blockIdx.x * I8_BN;
  constexpr int TILE = I8_BM * I8_BK;  // bytes per operand tile
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(I8_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < I8_ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int nk = K / I8_BK;
  uint32_t phase[I8_ST] = {0, 0};
  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt % I8_ST;
    if (kt >= I8_ST) {  // the MMAs that read this stage two iterations ago must be done
      mbar_wait(smem_u32(&mbar[st]), phase[st]);
      phase[st] ^= 1;
    }
    uint8_t* sa = sm + st * 2 * TILE;
    uint8_t* sb = sa + TILE;
    const int k0 = kt * I8_BK;
#pragma unroll 4
    for (int c = tid; c < I8_BM * 8; c += I8_T) {
      const int r = c >> 3, ch = c & 7;
      const int sw = (r * 128) + ((ch ^ (r & 7)) << 4);
      *reinterpret_cast<uint4*>(sa + sw) =
          __ldg(reinterpret_cast<const uint4*>(A + (long long)(m0 + r) * K + k0 + (ch << 4)));
      *reinterpret_cast<uint4*>(sb + sw) =
          __ldg(reinterpret_cast<const uint4*>(B + (long long)(n0 + r) * K + k0 + (ch << 4)));
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
#pragma unroll
      for (int kk = 0; kk < I8_BK / 32; ++kk)
        mma_i8(tmem, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), (kt | kk) != 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&mbar[st])));
    }
    __syncwarp();
  }
  // drain: the last commit of each stage
  for (int s = 0; s < I8_ST && s < nk; ++s) {
    const int st = (nk - 1 - s) % I8_ST;
    mbar_wait(smem_u32(&mbar[st]), phase[st]);
    phase[st] ^= 1;
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int j = 0; j < I8_BN; j += 16) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    int* out = C + (long long)row * N + n0 + j;
#pragma unroll
    for (int q = 0; q < 16; q += 4)
      *reinterpret_cast<int4*>(out + q) = make_int4((int)v[q], (int)v[q + 1], (int)v[q + 2], (int)v[q + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(I8_BN));
}

// ---- TMA-fed, warp-specialized variant: 128 x 256 tiles, TS-stage ring of full/empty mbarriers.
// Thread 0 (warp 0) is the TMA producer, thread 32 (warp 1) issues the MMAs; all four warps run
// the epilogue (TMEM lanes 32w..32w+31 belong to warp w).
constexpr int TB_M = 128, TB_N = 256, TB_K = 128, TS = 4;
constexpr uint32_t kIdescI8N256 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TB_N >> 3) << 17) |
                                  ((uint32_t)(TB_M >> 4) << 24);

__device__ __forceinline__ void mma_i8_n256(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescI8N256), "r"(acc));
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) i8gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                                                           const __grid_constant__ CUtensorMap tmB, int M, int N,
                                                           int K, int* __restrict__ C) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[TS], empty[TS], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * TB_M, n0 = blockIdx.x * TB_N;
  constexpr int ABYTES = TB_M * TB_K, BBYTES = TB_N * TB_K, SBYTES = ABYTES + BBYTES;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(TB_N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < TS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int nk = K / TB_K;
  // warps 0 and 1: lane 0 works, the other lanes park in __syncwarp (see the Ozaki kernel)
  if (warp == 0 && lane == 0) {
    // producer
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TS;
      if (kt >= TS) mbar_wait(smem_u32(&empty[s]), ((kt / TS) - 1) & 1);
      const uint32_t fb = smem_u32(&full[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fb), "r"(SBYTES) : "memory");
      const uint32_t sa = smem_u32(sm + s * SBYTES);
      tma_load_2d(sa, &tmA, kt * TB_K, m0, fb);
      tma_load_2d(sa + ABYTES, &tmB, kt * TB_K, n0, fb);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % TS;
      mbar_wait(smem_u32(&full[s]), (kt / TS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t a0 = smem_u32(sm + s * SBYTES), b0 = a0 + ABYTES;
#pragma unroll
      for (int kk = 0; kk < TB_K / 32; ++kk)
        mma_i8_n256(tmem, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), (kt | kk) != 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&empty[s])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        smem_u32(&done)));
  }
  __syncwarp();
  mbar_wait(smem_u32(&done), 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const int row = m0 + warp * 32 + lane;
#pragma unroll 1
  for (int j = 0; j < TB_N; j += 16) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    int* out = C + (long long)row * N + n0 + j;
#pragma unroll
    for (int q = 0; q < 16; q += 4)
      *reinterpret_cast<int4*>(out + q) = make_int4((int)v[q], (int)v[q + 1], (int)v[q + 2], (int)v[q + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TB_N));
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D int8 K-major operand (rows x K, row stride K bytes), box 128 bytes x box_rows, 128B swizzle
bool make_tmap(CUtensorMap* tm, const void* ptr, int rows, int K, int box_rows) {
  auto enc = tmap_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// C (int32 M x N) = A (int8 M x K) B (int8 N x K)^T, all row-major; M, N multiples of 128, K of 128.
TTB_API int ttb_i8gemm(void* stream, int M, int N, int K, const void* A, const void* B, int* C) {
  if (M % I8_BM || N % I8_BN || K % I8_BK || M <= 0 || N <= 0 || K <= 0) return TTB_EARG;
  static int variant = -1;
  if (variant < 0) {
    const char* e = getenv("TTB_I8GEMM");
    variant = (e && e[0] == 's') ? 0 : 1;  // s: synchronous-load kernel
  }
  if (variant == 1 && N % TB_N == 0) {
    CUtensorMap ta, tb;
    if (make_tmap(&ta, A, M, K, TB_M) && make_tmap(&tb, B, N, K, TB_N)) {
      const size_t smem = (size_t)TS * (TB_M + TB_N) * TB_K + 1024;
      static bool cfg2 = false;
      if (!cfg2) {
        cudaFuncSetAttribute(i8gemm_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cfg2 = true;
      }
      dim3 grid(N / TB_N, M / TB_M);
      i8gemm_tma_kernel<<<grid, 128, smem, as_stream(stream)>>>(ta, tb, M, N, K, C); ttb_count();
      return ttb_last_error();
    }
  }
  const size_t smem = (size_t)I8_ST * 2 * I8_BM * I8_BK + 1024;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(i8gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = true;
  }
  dim3 grid(N / I8_BN, M / I8_BM);
  i8gemm_kernel<<<grid, I8_T, smem, as_stream(stream)>>>(M, N, K, reinterpret_cast<const int8_t*>(A),
                                                         reinterpret_cast<const int8_t*>(B), C); ttb_count();
  return ttb_last_error();
}
