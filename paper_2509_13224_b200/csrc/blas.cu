// FP64 dense building blocks: DMMA GEMM, N-d permute, deterministic reductions.
//
// The GEMM is the contraction engine for every TT core product (TT-matvec,
// rounding carries, AMEn environments). It issues FP64 tensor-core MMAs
// (mma.sync m8n8k4 .f64 -> SASS DMMA) from shared-memory tiles filled with
// cp.async (LDGSTS) in a two-stage pipeline.
#include "common.cuh"
#include <stdlib.h>

long long g_ttb_launches = 0;

TTB_API long long ttb_launch_count(int reset) {
  long long v = __atomic_load_n(&g_ttb_launches, __ATOMIC_RELAXED);
  if (reset) __atomic_store_n(&g_ttb_launches, 0LL, __ATOMIC_RELAXED);
  return v;
}

namespace {

constexpr int kKcAlign = 32;  // split-K chunk alignment (multiple of every tile depth)
// tile depth: 32 for the 128 x 128 tiles (fewer barriers per K; measured +4%), 16 elsewhere
template <int BM, int BN>
constexpr int tile_bk() { return (BM == 128 && BN == 128) ? 32 : 16; }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct GemmArgs {
  int M, N, K;
  double alpha, beta;
  const double* A;
  long long lda, sA;
  int tA;
  const double* B;
  long long ldb, sB;
  int tB;
  double* C;
  long long ldc, sC;
  int split;  // split-K: blockIdx.z indexes K chunks of length Kc, partials to C + z*sC
  int Kc;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// Shared-memory tile layouts follow the global contiguity of each operand, so every
// global->shared copy is a contiguous (8 or 16 byte) cp.async and fragment reads are
// conflict-free (pitches chosen so a warp's 32 x 8 B fragment read is exactly two wavefronts):
//   A !tA : As[m][k] pitch BK+4     A tA : As[k][m] pitch BM+8
//   B !tB : Bs[k][n] pitch BN+8     B tB : Bs[n][k] pitch BK+4
template <int BM, int BN, int WM, int WN, int TA, int TB, int VEC, int STAGES, int CI>
__global__ void __launch_bounds__(WM* WN * 32) dgemm_kernel(GemmArgs g) {
  constexpr int T = WM * WN * 32;
  constexpr int BK = tile_bk<BM, BN>();
  constexpr int ASZ = TA ? BK * (BM + 8) : BM * (BK + 4);
  constexpr int BSZ = TB ? BN * (BK + 4) : BK * (BN + 8);
  constexpr int MT = BM / WM / 8, NT = BN / WN / 8;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;
  double* Bs = sm + STAGES * ASZ;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  // CI (short-K read-modify-write updates): M tiles fastest, so the CTAs sharing one B tile run
  // together and B is fetched from HBM once
  const int bm0 = (CI ? blockIdx.x : blockIdx.y) * BM, bn0 = (CI ? blockIdx.y : blockIdx.x) * BN;
  const long long bz = blockIdx.z;
  const double* A;
  const double* B;
  double* C = g.C + bz * g.sC;
  const int M = g.M, N = g.N;
  int K;
  if (g.split) {
    const long long kb = bz * g.Kc;
    K = (int)min((long long)g.Kc, (long long)g.K - kb);
    A = g.A + (TA ? kb * g.lda : kb);
    B = g.B + (TB ? kb : kb * g.ldb);
  } else {
    K = g.K;
    A = g.A + bz * g.sA;
    B = g.B + bz * g.sB;
  }

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load = [&](int kt, int st) {
    const int k0 = kt * BK;
    double* as = As + st * ASZ;
    double* bs = Bs + st * BSZ;
    // A tile: BM x BK
    {
      constexpr int CONT = TA ? BM : BK;   // contiguous extent in global
      constexpr int OUTER = TA ? BK : BM;
      constexpr int V = VEC;                // doubles per copy
      constexpr int PER = CONT / V;
#pragma unroll
      for (int e0 = 0; e0 < OUTER * PER; e0 += T) {
        const int e = e0 + tid;
        if (OUTER * PER % T != 0 && e >= OUTER * PER) break;
        const int o = e / PER, c = (e % PER) * V;
        int m, k;
        if (TA) { k = o; m = c; } else { m = o; k = c; }
        const int gm = bm0 + m, gk = k0 + k;
        double* dst = TA ? (as + k * (BM + 8) + m) : (as + m * (BK + 4) + k);
        const int rowok = TA ? (gk < K) : (gm < M);
        const int lim = TA ? (M - gm) : (K - gk);  // elements available along the contiguous dim
        const int avail = rowok ? (lim >= V ? V : (lim > 0 ? lim : 0)) : 0;
        const double* src = avail ? (TA ? A + (long long)gk * g.lda + gm : A + (long long)gm * g.lda + gk) : A;
        if (V == 2) cp_async16(dst, src, avail * 8);
        else cp_async8(dst, src, avail > 0);
      }
    }
    // B tile: BK x BN
    {
      constexpr int CONT = TB ? BK : BN;
      constexpr int OUTER = TB ? BN : BK;
      constexpr int V = VEC;
      constexpr int PER = CONT / V;
#pragma unroll
      for (int e0 = 0; e0 < OUTER * PER; e0 += T) {
        const int e = e0 + tid;
        if (OUTER * PER % T != 0 && e >= OUTER * PER) break;
        const int o = e / PER, c = (e % PER) * V;
        int n, k;
        if (TB) { n = o; k = c; } else { k = o; n = c; }
        const int gn = bn0 + n, gk = k0 + k;
        double* dst = TB ? (bs + n * (BK + 4) + k) : (bs + k * (BN + 8) + n);
        const int rowok = TB ? (gn < N) : (gk < K);
        const int lim = TB ? (K - gk) : (N - gn);
        const int avail = rowok ? (lim >= V ? V : (lim > 0 ? lim : 0)) : 0;
        const double* src = avail ? (TB ? B + (long long)gn * g.ldb + gk : B + (long long)gk * g.ldb + gn) : B;
        if (V == 2) cp_async16(dst, src, avail * 8);
        else cp_async8(dst, src, avail > 0);
      }
    }
  };

  const int nk = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_async_commit();
  }
  if (CI) {
    // short-K read-modify-write updates: fetch C while the first operand stages are in flight
    const double f = g.beta * g.alpha;  // == beta / alpha for alpha = +-1
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int m = bm0 + wm * (BM / WM) + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int n = bn0 + wn * (BN / WN) + j * 8 + (lane & 3) * 2;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (m < M && n + h < N) acc[i][j][h] = f * __ldg(C + (long long)m * g.ldc + n + h);
      }
    }
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load(nxt, nxt % STAGES);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * ASZ;
    const double* bs = Bs + (kt % STAGES) * BSZ;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MT], bf[NT];
      const int kr = kk + (lane & 3);
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int mr = wm * (BM / WM) + i * 8 + (lane >> 2);
        af[i] = TA ? as[kr * (BM + 8) + mr] : as[mr * (BK + 4) + kr];
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int nc = wn * (BN / WN) + j * 8 + (lane >> 2);
        bf[j] = TB ? bs[nc * (BK + 4) + kr] : bs[kr * (BN + 8) + nc];
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int m = bm0 + wm * (BM / WM) + i * 8 + (lane >> 2);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int n = bn0 + wn * (BN / WN) + j * 8 + (lane & 3) * 2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (n + h < N) {
          double* c = C + (long long)m * g.ldc + n + h;
          double v = g.alpha * acc[i][j][h];
          if (!g.split && !CI && g.beta != 0.0) v += g.beta * *c;
          *c = v;
        }
      }
    }
  }
}

template <int BM, int BN, int WM, int WN, int TA, int TB, int VEC, int CI>
int launch_gemm_t(const GemmArgs& g, int batch, cudaStream_t st) {
  constexpr int STAGES = 3;
  constexpr int T = WM * WN * 32;
  constexpr int BK = tile_bk<BM, BN>();
  constexpr int ASZ = TA ? BK * (BM + 8) : BM * (BK + 4);
  constexpr int BSZ = TB ? BN * (BK + 4) : BK * (BN + 8);
  const size_t smem = (size_t)STAGES * (ASZ + BSZ) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(dgemm_kernel<BM, BN, WM, WN, TA, TB, VEC, STAGES, CI>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  dim3 grid = CI ? dim3(ceil_div(g.M, BM), ceil_div(g.N, BN), batch) : dim3(ceil_div(g.N, BN), ceil_div(g.M, BM), batch);
  dgemm_kernel<BM, BN, WM, WN, TA, TB, VEC, STAGES, CI><<<grid, T, smem, st>>>(g); ttb_count();
  return ttb_last_error();
}

template <int BM, int BN, int WM, int WN, int CI = 0>
int launch_gemm(const GemmArgs& g, int batch, cudaStream_t st) {
  // 16-byte copies when both operands' rows (and batch strides) keep 16 B alignment
  const bool vec = ((g.lda & 1) == 0) && ((g.ldb & 1) == 0) && ((((uintptr_t)g.A) & 15) == 0) &&
                   ((((uintptr_t)g.B) & 15) == 0) && ((g.sA & 1) == 0) && ((g.sB & 1) == 0) &&
                   (!g.split || (g.Kc & 1) == 0);
  const int key = (g.tA ? 1 : 0) | (g.tB ? 2 : 0) | (vec ? 4 : 0);
  switch (key) {
    case 0: return launch_gemm_t<BM, BN, WM, WN, 0, 0, 1, CI>(g, batch, st);
    case 1: return launch_gemm_t<BM, BN, WM, WN, 1, 0, 1, CI>(g, batch, st);
    case 2: return launch_gemm_t<BM, BN, WM, WN, 0, 1, 1, CI>(g, batch, st);
    case 3: return launch_gemm_t<BM, BN, WM, WN, 1, 1, 1, CI>(g, batch, st);
    case 4: return launch_gemm_t<BM, BN, WM, WN, 0, 0, 2, CI>(g, batch, st);
    case 5: return launch_gemm_t<BM, BN, WM, WN, 1, 0, 2, CI>(g, batch, st);
    case 6: return launch_gemm_t<BM, BN, WM, WN, 0, 1, 2, CI>(g, batch, st);
    default: return launch_gemm_t<BM, BN, WM, WN, 1, 1, 2, CI>(g, batch, st);
  }
}

// C += alpha A B for a long, short-K product (WY trailing updates: M <= ~1024 rows of C_rm,
// K <= 128, N ~ 1e6; alpha = +-1, beta = 1). Persistent CTAs: each keeps its 64 x K block of A
// resident in shared memory and walks N tiles of WU_BN columns; B flows through a WU_S-stage ring
// of WU_KC-deep k-chunks (cp.async), continuous across tiles, and the next C tile is prefetched
// into registers while the current one is multiplied. 2 x WN warps.
constexpr int WU_BM = 64, WU_KMAX = 128;
constexpr int WU_LDA = WU_KMAX + 4;

template <int WU_BN, int WU_KC, int WU_S, int WN>
__global__ void __launch_bounds__(64 * WN, 1) wy_update_kernel(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                            long long lda, const double* __restrict__ B, long long ldb,
                                                            double* C, long long ldc) {
  constexpr int WU_LDB = WU_BN + 8;
  constexpr int WU_T = 64 * WN;  // 2 x WN warps
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                        // [WU_BM][WU_LDA]
  double* Bs = sm + WU_BM * WU_LDA;       // [WU_S][WU_KC][WU_LDB]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int bm0 = blockIdx.x * WU_BM;
  const int ntn = (N + WU_BN - 1) / WU_BN;
  constexpr int WNC = WU_BN / WN;  // warp tile columns
  const int nkc = (K + WU_KC - 1) / WU_KC;  // k-chunks per tile
  for (int e = tid; e < WU_BM * (WU_KMAX / 2); e += WU_T) {
    const int m = e / (WU_KMAX / 2), k = (e % (WU_KMAX / 2)) * 2;
    const int gm = bm0 + m;
    const int avail = (gm < M) ? max(0, min(2, K - k)) : 0;
    cp_async16(As + m * WU_LDA + k, avail ? A + (long long)gm * lda + k : A, avail * 8);
  }
  // my tiles: tn = blockIdx.y + i * gridDim.y; global chunk g -> (tile i = g / nkc, chunk g % nkc)
  const int my_tiles = (ntn - (int)blockIdx.y + (int)gridDim.y - 1) / (int)gridDim.y;
  const int nchunks = my_tiles > 0 ? my_tiles * nkc : 0;
  auto load_chunk = [&](int g) {
    if (g < nchunks) {
      const int tn = blockIdx.y + (g / nkc) * gridDim.y, kc = g % nkc;
      double* bs = Bs + (g % WU_S) * (WU_KC * WU_LDB);
      const int bn0 = tn * WU_BN, k0 = kc * WU_KC;
#pragma unroll
      for (int e0 = 0; e0 < WU_KC * (WU_BN / 2); e0 += WU_T) {
        const int e = e0 + tid;
        const int k = e / (WU_BN / 2), n = (e % (WU_BN / 2)) * 2;
        const int gn = bn0 + n, gk = k0 + k;
        const int avail = (gk < K) ? max(0, min(2, N - gn)) : 0;
        cp_async16(bs + k * WU_LDB + n, avail ? B + (long long)gk * ldb + gn : B, avail * 8);
      }
    }
    cp_async_commit();
  };
  constexpr int MT = 4, NT = WNC / 8;
  auto load_c = [&](int tn, double (&c)[MT][NT][2]) {
    const int bn0 = tn * WU_BN;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int m = bm0 + wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int n = bn0 + wn * WNC + j * 8 + (lane & 3) * 2;
        if (m < M && n + 1 < N) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(C + (long long)m * ldc + n));
          c[i][j][0] = v.x; c[i][j][1] = v.y;
        } else {
          c[i][j][0] = (m < M && n < N) ? C[(long long)m * ldc + n] : 0.0;
          c[i][j][1] = 0.0;
        }
      }
    }
  };
  // prologue: A block + chunks 0 .. S-2 (A rides in the first group)
  load_chunk(0);
#pragma unroll
  for (int g = 1; g < WU_S - 1; ++g) load_chunk(g);
  double cn[MT][NT][2], acc[MT][NT][2];
  if (my_tiles > 0) load_c(blockIdx.y, cn);
  for (int g = 0; g < nchunks; ++g) {
    const int kc = g % nkc;
    const int tn = blockIdx.y + (g / nkc) * gridDim.y;
    cp_async_wait<WU_S - 2>();
    __syncthreads();
    load_chunk(g + WU_S - 1);
    if (kc == 0) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          acc[i][j][0] = alpha * cn[i][j][0];  // exact for alpha = +-1: result = alpha (alpha C + A B)
          acc[i][j][1] = alpha * cn[i][j][1];
        }
      const int tnext = tn + gridDim.y;
      if (tnext < ntn) load_c(tnext, cn);
    }
    const double* bs = Bs + (g % WU_S) * (WU_KC * WU_LDB);
    // 16-deep steps (zero-filled beyond K): all fragments of a step are loaded before its MMAs
    const int kend = min(WU_KC, ((K + 15) & ~15) - kc * WU_KC);
    const double* as = As + (wm * 32 + (lane >> 2)) * WU_LDA + kc * WU_KC + (lane & 3);
    const double* bsl = bs + (lane & 3) * WU_LDB + wn * WNC + (lane >> 2);
    for (int kb = 0; kb < kend; kb += 16) {
      double af[4][MT], bf[4][NT];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int i = 0; i < MT; ++i) af[q][i] = as[i * 8 * WU_LDA + kb + 4 * q];
#pragma unroll
        for (int j = 0; j < NT; ++j) bf[q][j] = bsl[(kb + 4 * q) * WU_LDB + j * 8];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[q][i], bf[q][j]);
    }
    if (kc == nkc - 1) {
      const int bn0 = tn * WU_BN;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int m = bm0 + wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int n = bn0 + wn * WNC + j * 8 + (lane & 3) * 2;
          const double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
          if (m < M && n + 1 < N) {
            __stcs(reinterpret_cast<double2*>(C + (long long)m * ldc + n), make_double2(v0, v1));
          } else if (m < M && n < N) {
            C[(long long)m * ldc + n] = v0;
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

template <int BN, int KC, int S, int WN>
int launch_wy_update_t(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
                       double* C, long long ldc, cudaStream_t st) {
  const size_t smem = (size_t)(WU_BM * WU_LDA + S * KC * (BN + 8)) * sizeof(double);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(wy_update_kernel<BN, KC, S, WN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = true;
  }
  const int mt = (M + WU_BM - 1) / WU_BM;
  const int ntn = (N + BN - 1) / BN;
  static const int sms = getenv("TTB_WY_SMS") ? atoi(getenv("TTB_WY_SMS")) : ttb_num_sms();
  int gy = sms / mt;
  if (gy < 1) gy = 1;
  if (gy > ntn) gy = ntn;
  wy_update_kernel<BN, KC, S, WN><<<dim3(mt, gy), 64 * WN, smem, st>>>(M, N, K, alpha, A, lda, B, ldb, C, ldc);
  ttb_count();
  return ttb_last_error();
}

int launch_wy_update(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
                     double* C, long long ldc, cudaStream_t st) {
  // 64 x 64 tiles, whole-K B tiles double-buffered, 2 x 4 warps (measured best of the
  // 128-wide / k-chunk-ring / 4-warp variants on the 896 x 1M x 128 update)
  return launch_wy_update_t<64, 128, 2, 4>(M, N, K, alpha, A, lda, B, ldb, C, ldc, st);
}

__global__ void scale_kernel(long long n, double beta, double* C, long long ldc, int M, int N, long long sC) {
  // C = beta*C over an M x N (row-major, ldc) block per batch (used when K == 0)
  long long b = blockIdx.y;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    long long m = e / N, c = e % N;
    double* p = C + b * sC + m * ldc + c;
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

// C[r, c] = alpha * sum_k A[r, k] B[k, c] + beta * C[r, c] for small K (<= 32): every thread owns one
// column c of C and keeps B[:, c] in registers; the rows of A are staged in shared memory and read
// as broadcasts (one LDS.128 per two k), so the pass is bound by streaming C once through HBM.
template <int KT>
__global__ void __launch_bounds__(128) lowrank_update_kernel(int M, int N, int K, double alpha,
                                                             const double* __restrict__ A, long long lda,
                                                             const double* __restrict__ B, long long ldb,
                                                             double beta, double* C, long long ldc) {
  constexpr int RB = 32;  // rows of A staged per round
  __shared__ __align__(16) double As[RB][KT];
  const int c = blockIdx.x * 128 + threadIdx.x;
  double bk[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) bk[k] = (c < N && k < K) ? B[(long long)k * ldb + c] : 0.0;
  for (int r0 = 0; r0 < M; r0 += RB) {
    const int rn = min(RB, M - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < RB * KT; e += 128) {
      const int r = e / KT, k = e % KT;
      As[r][k] = (r < rn && k < K) ? A[(long long)(r0 + r) * lda + k] : 0.0;
    }
    __syncthreads();
    if (c < N) {
      for (int rr0 = 0; rr0 < rn; rr0 += 8) {  // 8 independent loads of C in flight
        double cv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          cv[u] = (beta != 0.0 && rr0 + u < rn) ? C[(long long)(r0 + rr0 + u) * ldc + c] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (rr0 + u < rn) {
            const double2* ar = reinterpret_cast<const double2*>(As[rr0 + u]);
            double acc = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < KT / 2; ++k2) {
              const double2 av = ar[k2];
              acc += av.x * bk[2 * k2] + av.y * bk[2 * k2 + 1];
            }
            C[(long long)(r0 + rr0 + u) * ldc + c] = alpha * acc + beta * cv[u];
          }
        }
      }
    }
  }
}

__global__ void splitk_reduce(int M, int N, int S, const double* __restrict__ part, double alpha, double beta,
                              double* C, long long ldc) {
  long long tot = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += part[(long long)z * tot + e];
    double* c = C + (e / N) * ldc + (e % N);
    double v = alpha * s;
    if (beta != 0.0) v += beta * *c;
    *c = v;
  }
}

// TTB_WY=legacy keeps the short-K updates on the tiled GEMM (A/B testing)
bool wy_legacy() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TTB_WY");
    v = (e && e[0] == 'l') ? 1 : 0;
  }
  return v == 1;
}

// split-K partial sums: one buffer per stream (the blocked QR runs panel work on a second stream
// concurrently with the trailing updates). Growing a buffer synchronizes the device first.
struct ScratchSlot {
  cudaStream_t st;
  double* p;
  size_t bytes;
  unsigned long long last;
};
ScratchSlot g_scratch[4] = {};
unsigned long long g_scratch_clock = 0;

double* scratch(size_t bytes, cudaStream_t st) {
  ScratchSlot* slot = nullptr;
  for (auto& s : g_scratch)
    if (s.p && s.st == st) slot = &s;
  if (!slot) {
    for (auto& s : g_scratch)
      if (!s.p) { slot = &s; break; }
    if (!slot) {  // evict the least recently used stream's buffer
      slot = &g_scratch[0];
      for (auto& s : g_scratch)
        if (s.last < slot->last) slot = &s;
      cudaDeviceSynchronize();
      cudaFree(slot->p);
      slot->p = nullptr;
      slot->bytes = 0;
    }
    slot->st = st;
  }
  slot->last = ++g_scratch_clock;
  if (bytes > slot->bytes) {
    if (slot->p) { cudaDeviceSynchronize(); cudaFree(slot->p); }
    const size_t want = bytes + bytes / 2;
    if (cudaMalloc(&slot->p, want) != cudaSuccess) { slot->p = nullptr; slot->bytes = 0; return nullptr; }
    slot->bytes = want;
  }
  return slot->p;
}

// ---------------------------------------------------------------------------
struct PermArgs {
  int nd;
  long long out_dims[8];
  long long in_stride_for_out[8];  // input stride of the input axis that lands on output axis k
};

__global__ void permute_kernel(PermArgs a, long long total, const double* __restrict__ src, double* __restrict__ dst) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < total; j += (long long)gridDim.x * blockDim.x) {
    long long rem = j, off = 0;
#pragma unroll 8
    for (int k = a.nd - 1; k >= 0; --k) {
      long long c = rem % a.out_dims[k];
      rem /= a.out_dims[k];
      off += c * a.in_stride_for_out[k];
    }
    dst[j] = src[off];
  }
}

// out[b, c, r] = in[b, r, c] through a padded 32x32 shared-memory tile
__global__ void transpose_tile_kernel(long long Bt, long long R, long long C, const double* __restrict__ src,
                                      double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (long long b = blockIdx.z; b < Bt; b += gridDim.z) {
    const double* in = src + b * R * C;
    double* out = dst + b * R * C;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const long long r = r0 + y, c = c0 + threadIdx.x;
      if (r < R && c < C) tile[y][threadIdx.x] = in[r * C + c];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const long long c = c0 + y, r = r0 + threadIdx.x;
      if (r < R && c < C) out[c * R + r] = tile[threadIdx.x][y];
    }
    __syncthreads();
  }
}

// out[b, c, r, s] = in[b, r, c, s] for contiguous runs of S >= 8 doubles (coalesced along s)
__global__ void transpose_runs_kernel(long long total, long long R, long long C, long long S,
                                      const double* __restrict__ src, double* __restrict__ dst) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long s = e % S;
    long long t = e / S;
    const long long r = t % R;
    t /= R;
    const long long c = t % C;
    const long long b = t / C;
    dst[e] = src[((b * R + r) * C + c) * S + s];
  }
}

// deterministic two-level reductions ----------------------------------------
constexpr int RED_BLOCKS = 296;
constexpr int RED_THREADS = 256;

__global__ void dot_partial(long long n, const double* __restrict__ x, const double* __restrict__ y, double* part) {
  __shared__ double sm[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += x[i] * (y ? y[i] : x[i]);
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_final(int np, const double* part, double* out, int take_sqrt) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) *out = take_sqrt ? sqrt(s) : s;
}

}  // namespace

// per-stream scratch buffer for other translation units (tt.cu band GEMM workspaces)
double* ttb_scratch(size_t bytes, cudaStream_t st) { return scratch(bytes, st); }

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C, long long ldc,
                      long long sC, int batch);
int ozaki_gemm(cudaStream_t st, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
               const double* B, long long ldb, double beta, double* C, long long ldc, void* ws);
long long ozaki_ws_bytes(int M, int N, int K);
bool ozaki_shape_ok(int M, int N, int K);

// The Householder WY products of the tall QRs (qr.cu): W = C V^T with K = the long dimension and the
// trailing update C += alpha W2 V with K = 128. With TTB_OZAKI_QR=1, large tileable shapes (M N K >= 2^33)
// run as Ozaki-scheme FP64 on the int8 tensor cores (ozaki.cu; split-K with exact int64 level sums for
// long K, beta epilogue for the update).
int dgemm_wy(void* stream, int tB, int M, int N, int K, double alpha, const double* A, long long lda, const double* B,
             long long ldb, double beta, double* C, long long ldc) {
  // opt-in (TTB_OZAKI_QR=1): measured slower than DMMA for these low-intensity shapes (geqrf 1M x 1024:
  // 175 vs 115 ms) -- operand slicing moves ~30 bytes per element of C against 2 x 128 flops, and the
  // K = 128 updates are TMEM-drain bound
  static const bool on = [] {
    const char* e = getenv("TTB_OZAKI_QR");
    return e && e[0] == '1';
  }();
  if (on && (long long)M * N * K >= (1LL << 33) && ozaki_shape_ok(M, N, K)) {
    cudaStream_t st = as_stream(stream);
    void* ws = scratch((size_t)ozaki_ws_bytes(M, N, K), st);
    if (ws) return ozaki_gemm(st, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws);
  }
  return ttb_dgemm(stream, 0, tB, M, N, K, alpha, A, lda, 0, B, ldb, 0, beta, C, ldc, 0, 1);
}

static int ttb_dgemm_impl(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A,
                          long long lda, long long sA, const double* B, long long ldb, long long sB, double beta,
                          double* C, long long ldc, long long sC, int batch);

static bool mid96_tiles() {  // TTB_GEMM_N96=0 disables the 128x96 tiles (A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TTB_GEMM_N96");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

TTB_API int ttb_dgemm(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      long long sA, const double* B, long long ldb, long long sB, double beta, double* C,
                      long long ldc, long long sC, int batch) {
  static const bool log = getenv("TTB_GEMM_LOG") != nullptr;   // shape log of the large DMMA GEMMs (tools)
  if (log && 2.0 * M * N * (double)K * batch >= 1e10)
    fprintf(stderr, "ttb_gemm tA=%d tB=%d M=%d N=%d K=%d batch=%d\n", tA, tB, M, N, K, batch);
  const int rc = ttb_dgemm_impl(stream, tA, tB, M, N, K, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC, batch);
  if (ttb_debug_sync()) {
    const cudaError_t e = cudaStreamSynchronize(as_stream(stream));
    if (e != cudaSuccess)
      fprintf(stderr, "ttb debug: dgemm tA=%d tB=%d M=%d N=%d K=%d lda=%lld ldb=%lld ldc=%lld batch=%d failed: %d\n", tA, tB, M,
              N, K, lda, ldb, ldc, batch, (int)e);
  }
  return rc;
}

static int ttb_dgemm_impl(void* stream, int tA, int tB, int M, int N, int K, double alpha, const double* A,
                          long long lda, long long sA, const double* B, long long ldb, long long sB, double beta,
                          double* C, long long ldc, long long sC, int batch) {
  if (M < 0 || N < 0 || K < 0 || batch < 0) return TTB_EARG;
  if (M == 0 || N == 0 || batch == 0) return TTB_OK;
  cudaStream_t st = as_stream(stream);
  if (K == 0) {
    long long n = (long long)M * N;
    dim3 grid(ceil_div(n, 256) > 1024 ? 1024 : ceil_div(n, 256), batch);
    scale_kernel<<<grid, 256, 0, st>>>(n, beta, C, ldc, M, N, sC); ttb_count();
    return ttb_last_error();
  }
  if (!tA && !tB && batch == 1 && K <= 32 && N >= 2048) {
    // low-rank update of a long matrix (WY panel updates): memory-bound, one coalesced RMW pass
    dim3 grid(ceil_div(N, 128));
    if (K <= 16)
      lowrank_update_kernel<16><<<grid, 128, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    else
      lowrank_update_kernel<32><<<grid, 128, 0, st>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
    ttb_count();
    return ttb_last_error();
  }
  GemmArgs g{M, N, K, alpha, beta, A, lda, sA, tA, B, ldb, sB, tB, C, ldc, sC, 0, 0};
  // alpha = +-1, beta != 0: the short-K path starts its accumulators at (beta/alpha) C (CI kernels)
  const bool cinit = beta != 0.0 && (alpha == 1.0 || alpha == -1.0);
  long long work = (long long)M * N * batch;
  // (N in [96, 128) stays on 64x64 tiles: measured faster than 128x128 for the banded-operator GEMMs,
  // 31.0 vs 26.8 TF/s at the configs[3] local shape even with even (16-byte) strides)
  const bool big = (work >= (long long)ttb_num_sms() * 128 * 128 * 2 || K >= 8192) && M >= 128 && N >= 128;
  const bool narrow = !big && N <= 32 && M >= 48;  // thin outputs (WY products over panel widths)
  const long long tiles = big ? (long long)ceil_div(M, 128) * ceil_div(N, 128) * batch
                        : narrow ? (long long)ceil_div(M, 128) * ceil_div(N, 32) * batch
                                 : (long long)ceil_div(M, 64) * ceil_div(N, 64) * batch;
  if (batch == 1 && tiles < ttb_num_sms() && K >= 1024) {
    // split-K: chunks filling (not exceeding) two waves of 148 SMs, each chunk >= 256 deep,
    // deterministic reduction
    long long S = 2LL * ttb_num_sms() / tiles;
    long long maxS = K / 256;
    if (S > maxS) S = maxS;
    if (S > 1) {
      int Kc = (int)(((K + S - 1) / S + kKcAlign - 1) / kKcAlign * kKcAlign);
      S = (K + Kc - 1) / Kc;
      double* part = scratch((size_t)S * M * N * sizeof(double), st);
      if (!part) return (int)cudaErrorMemoryAllocation;
      GemmArgs p = g;
      p.alpha = 1.0; p.beta = 0.0; p.C = part; p.ldc = N; p.sC = (long long)M * N; p.split = 1; p.Kc = Kc;
      int rc = big ? launch_gemm<128, 128, 2, 4>(p, (int)S, st)
                   : narrow ? launch_gemm<128, 32, 4, 1>(p, (int)S, st) : launch_gemm<64, 64, 2, 2>(p, (int)S, st);
      if (rc) return rc;
      long long tot = (long long)M * N;
      int blocks = ceil_div(tot, 256);
      if (blocks > ttb_num_sms() * 8) blocks = ttb_num_sms() * 8;
      splitk_reduce<<<blocks, 256, 0, st>>>(M, N, (int)S, part, alpha, beta, C, ldc); ttb_count();
      return ttb_last_error();
    }
  }
  if (!tA && !tB && batch == 1 && K <= WU_KMAX && N >= 8192 && M >= 32 && beta == 1.0 && cinit &&
      !wy_legacy() && ((lda | ldb | ldc) & 1) == 0 && ((((uintptr_t)A) | ((uintptr_t)B) | ((uintptr_t)C)) & 15) == 0)
    return launch_wy_update(M, N, K, alpha, A, lda, B, ldb, C, ldc, st);
  // short-K updates of a long C (WY trailing updates): 128x64 tiles, ~120 registers -> 2 CTAs/SM so
  // one CTA's epilogue read-modify-write overlaps the other's main loop
  if (big && K <= 256 && N >= 4096)
    return cinit ? launch_gemm<128, 64, 4, 2, 1>(g, batch, st) : launch_gemm<128, 64, 4, 2>(g, batch, st);
  if (big) return launch_gemm<128, 128, 2, 4>(g, batch, st);
  if (narrow) return launch_gemm<128, 32, 4, 1>(g, batch, st);
  // TT-rank-wide outputs (65 <= N <= 96, e.g. the AMEn local operator's phiR stage): one 96-wide
  // column tile instead of two 64-wide ones (which would be 50-75% full)
  if (N > 64 && N <= 96 && M >= 256 && work >= (long long)ttb_num_sms() * 128 * 96 && mid96_tiles())
    return launch_gemm<128, 96, 4, 2>(g, batch, st);
  return launch_gemm<64, 64, 2, 2>(g, batch, st);
}

// dst = permute(src): src has dims in_dims[0..nd) (row-major); output axis k is input axis perm[k].
TTB_API int ttb_permute(void* stream, int nd, const long long* in_dims, const int* perm, const double* src, double* dst) {
  if (nd < 1 || nd > 8) return TTB_EARG;
  PermArgs a;
  a.nd = nd;
  long long stride[8];
  long long s = 1;
  for (int k = nd - 1; k >= 0; --k) { stride[k] = s; s *= in_dims[k]; }
  long long total = s;
  for (int k = 0; k < nd; ++k) {
    if (perm[k] < 0 || perm[k] >= nd) return TTB_EARG;
    a.out_dims[k] = in_dims[perm[k]];
    a.in_stride_for_out[k] = stride[perm[k]];
  }
  if (total == 0) return TTB_OK;
  // fast path: perm = [prefix | B-group | A-group | suffix] of input [prefix | A | B | suffix]
  // -> out[b, c, r, s] = in[b, r, c, s]: coalesced run copies (S >= 8) or 32x32 smem tiles (S == 1)
  {
    int p0 = 0;
    while (p0 < nd && perm[p0] == p0) ++p0;
    int sfx = 0;
    while (sfx < nd - p0 && perm[nd - 1 - sfx] == nd - 1 - sfx) ++sfx;
    const int mid = nd - p0 - sfx;
    if (mid >= 2) {
      const int first = perm[p0];  // start of the B group in the input
      const int la = first - p0;   // length of A
      bool ok = la >= 1 && la < mid;
      for (int k = 0; ok && k < mid; ++k) {
        const int want = (k < mid - la) ? first + k : p0 + (k - (mid - la));
        ok = perm[p0 + k] == want;
      }
      if (ok) {
        long long Bt = 1, R = 1, Cc = 1, S = 1;
        for (int k = 0; k < p0; ++k) Bt *= in_dims[k];
        for (int k = p0; k < p0 + la; ++k) R *= in_dims[k];
        for (int k = p0 + la; k < nd - sfx; ++k) Cc *= in_dims[k];
        for (int k = nd - sfx; k < nd; ++k) S *= in_dims[k];
        cudaStream_t st = as_stream(stream);
        if (S == 1) {
          dim3 grid(ceil_div(Cc, 32), ceil_div(R, 32), (unsigned)(Bt < 65535 ? Bt : 65535));
          transpose_tile_kernel<<<grid, dim3(32, 8), 0, st>>>(Bt, R, Cc, src, dst); ttb_count();
          return ttb_last_error();
        }
        if (S >= 8) {
          int blocks = ceil_div(total, 256);
          if (blocks > ttb_num_sms() * 16) blocks = ttb_num_sms() * 16;
          transpose_runs_kernel<<<blocks, 256, 0, st>>>(total, R, Cc, S, src, dst); ttb_count();
          return ttb_last_error();
        }
      }
    }
  }
  int blocks = ceil_div(total, 256);
  if (blocks > ttb_num_sms() * 16) blocks = ttb_num_sms() * 16;
  permute_kernel<<<blocks, 256, 0, as_stream(stream)>>>(a, total, src, dst); ttb_count();
  return ttb_last_error();
}

// out[0] = x.y (y == NULL -> ||x||^2; take_sqrt -> ||x||). part: >= 296 doubles of scratch.
TTB_API int ttb_dot(void* stream, long long n, const double* x, const double* y, double* out, double* part,
                    int take_sqrt) {
  cudaStream_t st = as_stream(stream);
  int blocks = n <= 0 ? 1 : (ceil_div(n, RED_THREADS) < RED_BLOCKS ? ceil_div(n, RED_THREADS) : RED_BLOCKS);
  dot_partial<<<blocks, RED_THREADS, 0, st>>>(n, x, y, part); ttb_count();
  sum_final<<<1, 256, 0, st>>>(blocks, part, out, take_sqrt); ttb_count();
  return ttb_last_error();
}
