// FP64 GEMM emulated on the tcgen05 INT8 tensor cores (Ozaki scheme, error-free slicing).
//
// C (M x N) = A (M x K) B (K x N), FP64. Every row i of A is scaled by 2^-ea_i (ea_i = frexp
// exponent of max_k |a_ik|, so the scaled row lies in (-1, 1)) and cut into S = 7 balanced signed
// 8-bit slices,  a_ik = 2^ea_i sum_s sigma_s(i,k) 2^(-6-8s),  sigma_s in [-128, 127],
// the base-256 digits of the 54-bit integer round(a_ik 2^(54-ea_i)); B's columns likewise (exponents
// fb_j, slices tau_t, stored transposed: K-major). Then
//   C_ij = 2^(ea_i + fb_j) sum_{d<LEV} 2^(-12-8d) D_d(i, j),   D_d = sum_{s+t=d} A_s B_t^T,
// where every D_d is an exact int32 tcgen05 kind::i8 GEMM ((pairs per level) K 2^14 < 2^31 for
// K <= 4096). LEV = 8 keeps every product down to the 2^-54 level of the operands' slicing; the
// dropped levels weigh < 2^-60 K max|a_i| max|b_j|. Agreement with a DGEMM is at its own rounding
// level, normwise (tests/test_gpu_kernels.py). TTB_OZAKI_LEVELS=7 drops level 7 (28 products).
//
// Kernel: 128 x 64 output tiles, TMA (3-D maps over the slice stacks, 64-byte swizzle) into a
// 2-stage ring of full/empty mbarriers holding all 14 slice tiles of a 64-byte k step; one thread
// issues, per A slice s, MMAs of N = 64 nt against nt consecutive B slice tiles (the level
// accumulators s .. s+nt-1 are consecutive 64-column TMEM ranges), 10 MMAs per 32-byte k step for
// 34 slice products; the epilogue sums the levels in FP64 and writes C once through shared memory.
#include <vector>

#include "common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>

namespace {

constexpr int OZ_S = 7;                  // slices per operand
constexpr int OZ_M = 128;
constexpr int OZ_NONFINITE = 1 << 20;   // exponent of a row/column with an Inf/NaN maximum

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }


__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
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

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(mbar)
      : "memory");
}

// multicast variant: the box lands at the same shared-memory offset in every CTA of ctamask and signals
// the mbarrier at the same offset in each of them
__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t mbar,
                                               uint16_t ctamask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(mbar), "h"(ctamask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ---- all levels in one pass: 128 x 64 tiles, every k stage (64 bytes of K) holds all 7 A and all 7 B
// slices (84 KB, 2-stage ring, 64-byte swizzle), the 34 slice-pair MMAs accumulate into 8 TMEM
// accumulators of 64 columns (all 512), and C is written once.
#ifndef TTB_OZ_K
#define TTB_OZ_K 64
#endif
// k step per stage (bytes of K): 64 -> 64-byte swizzle, 2 stages of 84 KB (default); 32 -> 32-byte
// swizzle, 4 stages of 42 KB (measured slower: 28.1 vs 26.4 ms on 262144x4096x1024, Gram 38 vs 23 ms)
constexpr int OA_N = 64, OA_K = TTB_OZ_K, OA_ST = OA_K == 32 ? 4 : 2;
constexpr int OA_ABYTES = OZ_M * OA_K, OA_BBYTES = OA_N * OA_K;
constexpr int OA_SBYTES = OZ_S * (OA_ABYTES + OA_BBYTES);

// K-major, OA_K-byte swizzle (32 or 64): 8-row atoms of 8 OA_K bytes (SM100 layout type 6 / 4)
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(((8 * OA_K) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(OA_K == 32 ? 6 : 4) << 61;
  return d;
}

// s8 x s8 -> s32, M = 128, N = 64 nt (all slices are balanced signed digits)
__host__ __device__ constexpr uint32_t oa_idesc(int nt) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nt * OA_N >> 3) << 17) | ((uint32_t)(OZ_M >> 4) << 24);
}

// One 32-byte k step of every slice product of a tile. For A slice s the B slices t = 0..T_s-1
// (T_s = min(S, LEV - s)) are consecutive 64-row tiles in shared memory, i.e. one K-major operand of
// 64 T_s rows, and their products land in the level accumulators s..s+T_s-1, i.e. TMEM columns
// 64 s .. 64 (s + T_s): one MMA of N = 64 nt per chunk of <= 4 tiles (N <= 256) covers nt slice pairs
// and reads the A tile once for all of them. The MMAs that only touch not-yet-written levels (A slice 0,
// and for LEV 8 the (3, 4) product, level 7 alone) come first and overwrite (first = k step 0 of the
// tile), so the accumulators need no zeroing.
template <int LEV>
__device__ __forceinline__ void oz_issue(uint32_t tmem, uint64_t da, uint64_t db, int kk, bool first) {
  auto mma = [&](int sa, int t0, int nt, bool fresh) {
    mma_i8(tmem + (uint32_t)((sa + t0) * OA_N), da + (uint64_t)((sa * OA_ABYTES + kk * 32) >> 4),
           db + (uint64_t)((t0 * OA_BBYTES + kk * 32) >> 4), oa_idesc(nt), (fresh && first) ? 0u : 1u);
  };
  mma(0, 0, 4, true);
  mma(0, 4, 3, true);
  if (LEV == 8) mma(3, 4, 1, true);
#pragma unroll
  for (int sa = 1; sa < OZ_S; ++sa) {
    const int T = (LEV - sa < OZ_S) ? LEV - sa : OZ_S;
#pragma unroll
    for (int t0 = 0; t0 < T; t0 += 4) {
      if (LEV == 8 && sa == 3 && t0 == 4) continue;
      mma(sa, t0, T - t0 < 4 ? T - t0 : 4, false);
    }
  }
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

constexpr int OA_EPAD = 17;  // epilogue staging row (doubles) of a warp's 32 x 16 block

// Persistent, warp-specialized: warp 0 = TMA producer (lane 0), warp 1 = MMA issuer (lane 0), warps 2-9
// = epilogue (warp w reads TMEM lanes 32 (w % 4) ..). One 128 x 64 tile at a time in TMEM (all 512
// columns: 8 levels x 64); the producer runs ahead into the next tile's stages while the epilogue
// drains TMEM, and the epilogue's C write overlaps the next tile's MMAs (TMEM is released as soon as
// the level sums are in registers).
// Output of one work unit (a 128 x 64 tile over one K range): mode 0 out = x; mode 1 out + range * so
// = x (split-K partials, reduced by oz_reduce_kernel); mode 2 out = alpha x + beta out.
struct OzOut {
  double* out;
  long long ldo, so;
  double alpha, beta;
  int mode;
  int trilA;  // 1: A lower triangular (M == K, one K range): row block m0 stops at k = m0 + 128;
              // 2: B upper triangular (N == K, one K range): column block n0 stops at k = n0 + 64
  int mv, nv; // modes 0 / 2 of a padded product: only rows < mv and columns < nv are written (0: all)
  // mode 3 (TT-matvec core layout): row r = (a n + i) Rb + b, column c rd + d of the product go to
  // out[((a rc + c) n + i) Rb rd + b rd + d] (rd % 16 == 0, so a 16-column store segment has one c)
  int sn, sRb, src_, srd;
  // 1: tiles in row-block-fastest order (unit t -> row block t % (M / 128), column block t / (M / 128)):
  // few row blocks over a small A and a long B (C = carry x core, 1024 x 1M): the CTAs running together
  // then share B's column blocks through L2 instead of each row block re-reading the whole B stack
  int mfast;
};

// Banded batched mode (ttb_band_gemm_ozaki): batch i multiplies a K window of its group's A slice stack
// (group g = i / G holds the Tp blocks of batches gG .. gG+G-1 under one exponent per row) by its own B
// slices: units are (batch, 128 x 64 tile); A rows come from z = 7 g of the 3-D map at K offset
// (i - gG) Rin, B rows from i Np, C from out + i cstride with rows < X and columns < Rout written.
struct OzBand {
  int G, Rin /* K block per batch offset (padded) */, Mp, Np, Kp, X, Rout, nb;
  long long cstride;
};

constexpr int OZ_SUB = 64;

// tile t -> (m0, n0); sym: only the tiles touching the upper block triangle of a square output
// (column block >= 2 x row block), row by row
__device__ __forceinline__ void oz_tile(int t, int ntn, int sym, int& m0, int& n0) {
  if (!sym) {
    m0 = (t / ntn) * OZ_M;
    n0 = (t % ntn) * OA_N;
    return;
  }
  int mt = 0;
  while (t >= ntn - 2 * mt) {
    t -= ntn - 2 * mt;
    ++mt;
  }
  m0 = mt * OZ_M;
  n0 = (2 * mt + t) * OA_N;
}  // k steps (of 64) per TMEM accumulation: K <= 4096 keeps every level sum exact in int32

// CL = 2: 2-CTA clusters whose CTAs take consecutive units (same A rows, same K range, in lockstep); the A
// slice tiles are loaded once by rank 0 and multicast into both CTAs' shared memory, and every stage is
// released only when both CTAs' MMAs are done with it (empty barriers count one commit from each)
template <int LEV, bool LONGK, bool BAND = false, int CL = 1>  // LONGK: K ranges deeper than OZ_SUB k steps
__global__ void __launch_bounds__(320, 1) oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                                                        int kchunk, int ksplit, int tiles, int sym,
                                                        const int* __restrict__ ea,
                                                        const int* __restrict__ fb, const OzOut o,
                                                        const OzBand bd = OzBand{}) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[OA_ST], empty[OA_ST], tfull, tempty;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int s = 0; s < OA_ST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&empty[s])), "r"(CL));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&tfull)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" ::"r"(smem_u32(&tempty)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if constexpr (CL == 2) cluster_sync_all();   // peer barriers initialised before any multicast / commit
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const int crank = CL == 2 ? (int)(blockIdx.x & 1) : 0;
  // work unit u: K range u / tiles (kchunk deep), tile u % tiles (n fastest, so CTAs that run
  // together share the A rows); a range is accumulated in TMEM OZ_SUB k steps at a time
  const int ntn = (BAND ? bd.Np : N) / OA_N, units = BAND ? tiles * bd.nb : tiles * ksplit;
  // work unit -> output tile (m0, n0) and k-step range [kt0, kt1); banded mode: batch bi
  auto unit = [&](int u, int& m0, int& n0, int& kt0, int& kt1, int& bi) {
    if constexpr (BAND) {
      bi = u / tiles;
      const int t = u % tiles;
      m0 = (t / ntn) * OZ_M;
      n0 = (t % ntn) * OA_N;
      kt0 = 0;
      kt1 = bd.Kp / OA_K;
    } else {
      bi = 0;
      if (o.mfast) {
        const int t = u % tiles, ntm = M / OZ_M;
        m0 = (t % ntm) * OZ_M;
        n0 = (t / ntm) * OA_N;
      } else {
        oz_tile(u % tiles, ntn, sym, m0, n0);
      }
      if (o.trilA == 2) {
        // column block c of an upper-triangular B has c + 1 k steps: rotate the column order by the row
        // block, so the units a CTA takes (u, u + grid, ...) cycle through every depth instead of a
        // fixed residue class of c (148 = 4 mod 16: the deepest class did 10 k steps on average, the
        // mean is 8.5); a row block's tiles still run together and share its A rows
        n0 = (int)(((unsigned)(n0 / OA_N) + (unsigned)(m0 / OZ_M)) % (unsigned)ntn) * OA_N;
      }
      kt0 = (u / tiles) * (kchunk / OA_K);
      kt1 = min(min(K, (u / tiles + 1) * kchunk), o.trilA == 1 ? m0 + OZ_M : (o.trilA == 2 ? n0 + OA_N : K)) / OA_K;
    }
  };
  if (warp == 0) {
    if (lane == 0) {  // TMA producer: per stage one box of all 7 A slice tiles, one of all 7 B
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int m0, n0, kt0, kt1, bi;
        unit(u, m0, n0, kt0, kt1, bi);
        for (int kt = kt0; kt < kt1; ++kt, ++it) {
          const int st = it % OA_ST;
          if (it >= OA_ST) mbar_wait(smem_u32(&empty[st]), ((it / OA_ST) - 1) & 1);
          const uint32_t fbar = smem_u32(&full[st]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fbar), "r"(OA_SBYTES)
                       : "memory");
          const uint32_t base = smem_u32(sm + st * OA_SBYTES);
          if constexpr (BAND) {
            const int gi = bi / bd.G;
            if constexpr (CL == 2) {
              if (crank == 0)
                tma_load_3d_mc(base, &tmA, (bi - gi * bd.G) * bd.Rin + kt * OA_K, m0, OZ_S * gi, fbar, (uint16_t)3);
            } else {
              tma_load_3d(base, &tmA, (bi - gi * bd.G) * bd.Rin + kt * OA_K, m0, OZ_S * gi, fbar);
            }
            tma_load_3d(base + OZ_S * OA_ABYTES, &tmB, kt * OA_K, n0, OZ_S * bi, fbar);
          } else {
            if constexpr (CL == 2) {
              if (crank == 0) tma_load_3d_mc(base, &tmA, kt * OA_K, m0, 0, fbar, (uint16_t)3);
            } else {
              tma_load_3d(base, &tmA, kt * OA_K, m0, 0, fbar);
            }
            tma_load_3d(base + OZ_S * OA_ABYTES, &tmB, kt * OA_K, n0, 0, fbar);
          }
        }
      }
      if constexpr (CL == 2) {   // drain: every commit (own and peer) of the last stages has arrived
        for (int j = (it > OA_ST ? it - OA_ST : 0); j < it; ++j) mbar_wait(smem_u32(&empty[j % OA_ST]), (j / OA_ST) & 1);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int it = 0, g = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int m0, n0, kt0, kt1, bi;
        unit(u, m0, n0, kt0, kt1, bi);
        for (int ks = kt0; ks < kt1; ks += OZ_SUB, ++g) {
          if (g > 0) {  // the epilogue has the previous accumulation's level sums in registers
            mbar_wait(smem_u32(&tempty), (g - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
          }
          const int ke = min(kt1, ks + OZ_SUB);
          for (int kt = ks; kt < ke; ++kt, ++it) {
            const int st = it % OA_ST;
            mbar_wait(smem_u32(&full[st]), (it / OA_ST) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            const uint32_t a0 = smem_u32(sm + st * OA_SBYTES), b0 = a0 + OZ_S * OA_ABYTES;
            const uint64_t da = sw_desc(a0), db = sw_desc(b0);
#pragma unroll
            for (int kk = 0; kk < OA_K / 32; ++kk) oz_issue<LEV>(tmem, da, db, kk, kt == ks && kk == 0);
            if constexpr (CL == 2)
              asm volatile(
                  "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                      smem_u32(&empty[st])),
                  "h"((uint16_t)3));
            else
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                  smem_u32(&empty[st])));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              smem_u32(&tfull)));
        }
      }
    }
  } else {
    // epilogue, 8 warps: warp w reads TMEM lanes 32 (w % 4) .. (its 32 rows) and columns 32 h ..
    // (h = (w - 2) / 4) of every level. While TMEM is held only integer work runs: the level sums are
    // folded exactly into two int64 per column, hi = sum_{d<4} D_d 2^(8(3-d)) (|hi| < 2^51) and
    // lo = sum_{d>=4} D_d 2^(8(LEV-1-d)) (|lo| < 2^52.4 for K <= 4096), one IMAD.WIDE per level. TMEM is
    // released, then C = 2^e (hi 2^-36 + lo 2^-(12+8(LEV-1))), e = ea_i + fb_j, in one FMA (exact
    // products, a single rounding) and written through a per-warp 32 x 16 staging block, two rows of
    // 16 consecutive columns (128 bytes each) per store instruction.
    const int q = warp & 3, h = (warp - 2) >> 2;
    double* stg = reinterpret_cast<double*>(sm + OA_ST * OA_SBYTES) + (warp - 2) * 32 * OA_EPAD;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * 32);
    constexpr int LO_EXP = -12 - 8 * (LEV - 1);
    int g = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int m0, n0, kt0, kt1, bi;
      unit(u, m0, n0, kt0, kt1, bi);
      n0 += h * 32;
      const int my_ea = BAND ? ea[(bi / bd.G) * bd.Mp + m0 + q * 32 + lane] : ea[m0 + q * 32 + lane];
      const int my_fb = BAND ? fb[bi * bd.Np + n0 + lane] : fb[n0 + lane];  // column n0 + lane's exponent
      long long hi[32], lo[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) hi[c] = lo[c] = 0;
      for (int ks = kt0;;) {
        mbar_wait(smem_u32(&tfull), g & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll
        for (int d = 0; d < LEV; ++d) {
          const long long sh = 1LL << (d < 4 ? 8 * (3 - d) : 8 * (LEV - 1 - d));
#pragma unroll
          for (int gg = 0; gg < 2; ++gg) {  // 16 columns per load (10 warps: 168 registers per thread)
            uint32_t v[16];
            tmem_ld16(tq + (uint32_t)(d * OA_N + gg * 16), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              if (d < 4)
                hi[gg * 16 + c] += (long long)(int)v[c] * sh;
              else
                lo[gg * 16 + c] += (long long)(int)v[c] * sh;
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&tempty)) : "memory");
        ++g;
        ks += OZ_SUB;
        if (!LONGK || ks >= kt1) break;
      }
      const int cq = lane & 15, half = lane >> 4;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int cc = j * 16 + c;
          const int e = my_ea + __shfl_sync(0xffffffffu, my_fb, cc);
          double x;
          if (e >= OZ_NONFINITE)
            x = __longlong_as_double(0x7ff8000000000000LL);   // a non-finite operand row/column
          else if (e - 36 < 1024 && e + LO_EXP > -1023)
            x = fma((double)lo[cc], __longlong_as_double((long long)(e + LO_EXP + 1023) << 52),
                    (double)hi[cc] * __longlong_as_double((long long)(e - 36 + 1023) << 52));
          else
            x = ldexp(fma((double)lo[cc], __longlong_as_double((long long)(LO_EXP + 36 + 1023) << 52),
                          (double)hi[cc]), e - 36);
          stg[lane * OA_EPAD + c] = x;
        }
        __syncwarp();
        double* crow = o.out + (o.mode == 1 ? (long long)(u / tiles) * o.so : 0LL) + (long long)(m0 + q * 32) * o.ldo +
                       n0 + j * 16 + cq;
        if (!BAND && o.mode == 3) {
          const int col = n0 + j * 16 + cq;
          const int cc = col / o.srd, dd = col - cc * o.srd;
          const long long cb = (long long)cc * o.sn * o.sRb * o.srd + dd;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int rr = 2 * i + half;
            const int r = m0 + q * 32 + rr;
            const int b = r % o.sRb, ai = r / o.sRb;
            const int ii = ai % o.sn, a = ai / o.sn;
            o.out[(((long long)a * o.src_) * o.sn + ii) * o.sRb * o.srd + (long long)b * o.srd + cb] =
                stg[rr * OA_EPAD + cq];
          }
        } else if constexpr (BAND) {
          crow = o.out + (long long)bi * bd.cstride + (long long)(m0 + q * 32) * o.ldo + n0 + j * 16 + cq;
          if (n0 + j * 16 + cq < bd.Rout) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int rr = 2 * i + half;
              if (m0 + q * 32 + rr < bd.X) crow[(long long)rr * o.ldo] = stg[rr * OA_EPAD + cq];
            }
          }
        } else if (o.mv > 0) {   // padded product: rows >= mv / columns >= nv are padding
          if (n0 + j * 16 + cq < o.nv) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int rr = 2 * i + half;
              if (m0 + q * 32 + rr < o.mv) {
                const double y = o.alpha * stg[rr * OA_EPAD + cq];
                crow[(long long)rr * o.ldo] =
                    (o.mode != 2 || o.beta == 0.0) ? y : fma(o.beta, crow[(long long)rr * o.ldo], y);
              }
            }
          }
        } else if (o.mode == 2) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int rr = 2 * i + half;
            const double y = o.alpha * stg[rr * OA_EPAD + cq];
            crow[(long long)rr * o.ldo] = o.beta == 0.0 ? y : fma(o.beta, crow[(long long)rr * o.ldo], y);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int rr = 2 * i + half;
            crow[(long long)rr * o.ldo] = stg[rr * OA_EPAD + cq];
          }
        }
        __syncwarp();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if constexpr (CL == 2) cluster_sync_all();   // no CTA leaves while its peer may still signal it
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

// ---- slicing
// Non-finite operands: the row/column maxima propagate NaN (fmax would drop it) and a row or column
// whose maximum is Inf/NaN gets the exponent OZ_NONFINITE; every output that touches it is written
// as NaN (DGEMM would give Inf or NaN there), so an upstream breakdown is not hidden by the slicing.
__device__ __forceinline__ double oz_amax(double m, double x) {
  const double a = fabs(x);
  return (a > m || a != a) ? a : m;   // sticky NaN: NaN > m is false, and m stays NaN once it is
}
__device__ __forceinline__ int oz_exp_of(double m) {
  int ex = 0;
  if (!(m <= 1.7976931348623157e308)) return OZ_NONFINITE;   // Inf or NaN
  if (m > 0.0) frexp(m, &ex);
  return ex;
}

// exponent of the row maximum (frexp): one warp per row of a row-major (rows x K, ld) matrix
__global__ void oz_rowexp_kernel(int rows, int K, const double* __restrict__ X, long long ld, int* e) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  double m = 0.0;
  for (int k = lane; k < K; k += 32) m = oz_amax(m, X[(long long)w * ld + k]);
  for (int o = 16; o; o >>= 1) m = oz_amax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) e[w] = oz_exp_of(m);
}

// row maxima of a row-major (rows x K, ld) matrix with long rows: warp per (row, 8192-wide segment),
// atomicMax of the non-negative bit pattern (then oz_colexp_kernel)
__global__ void oz_rowmax_kernel(int rows, int K, const double* __restrict__ X, long long ld,
                                 unsigned long long* rmax) {
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int k0 = blockIdx.y * 8192, k1 = min(K, k0 + 8192);
  double m = 0.0;
  for (int k = k0 + lane; k < k1; k += 32) m = oz_amax(m, X[(long long)r * ld + k]);
  for (int o = 16; o; o >>= 1) m = oz_amax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMax(rmax + r, (unsigned long long)__double_as_longlong(m));
}

// C = alpha sum_s part[s] + beta C (fixed summation order: deterministic)
// C (M x N valid of the pM x pN partial layout) = alpha sum_s part[s] + beta C
__global__ void oz_reduce_kernel(int M, int N, int S, const double* __restrict__ part, double alpha, double beta,
                                 double* C, long long ldc, int pM, int pN) {
  const long long tot = (long long)M * N, ptot = (long long)pM * pN;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / N, j = e % N;
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc += part[(long long)s * ptot + i * pN + j];
    double* c = C + i * ldc + j;
    *c = beta == 0.0 ? alpha * acc : fma(beta, *c, alpha * acc);
  }
}

// exponent of the column maximum of a row-major (K x cols, ld) matrix: per-column atomicMax of the
// non-negative bit pattern, then frexp
__global__ void oz_colmax_kernel(int K, int cols, const double* __restrict__ X, long long ld,
                                 unsigned long long* cmax) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int k0 = blockIdx.y * 256, k1 = min(K, k0 + 256);
  double m = 0.0;
  for (int k = k0; k < k1; ++k) m = oz_amax(m, X[(long long)k * ld + c]);
  atomicMax(cmax + c, (unsigned long long)__double_as_longlong(m));
}

__global__ void oz_colexp_kernel(int cols, const unsigned long long* cmax, int* e) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  e[c] = oz_exp_of(__longlong_as_double((long long)cmax[c]));   // NaN's bit pattern is above Inf's
}

// Balanced base-256 digits of the 54-bit fixed-point value X = round(x 2^(54 - ex)) (|X| <= 2^54 - 1):
// X = sum_s sigma_s 2^(48 - 8s), every sigma_s in [-128, 127] (each byte above 127 borrows from the next
// digit up; the top digit stays within [-65, 65]), i.e. x = 2^ex sum_s sigma_s 2^(-6-8s) up to the single
// rounding of X. Integer arithmetic: a floor cascade in floating point loses the remainder of tiny values.
// sc = 2^(54 - ex) when that is a normal double (then x sc is exact, like ldexp), else 0 (use ldexp).
__device__ __forceinline__ double oz_scale_of(int ex) {
  const int p = 54 - ex;
  return (p > -1023 && p < 1024) ? __longlong_as_double((long long)(p + 1023) << 52) : 0.0;
}

// The digits of 4 values packed per plane: w[s] byte q = digit s of v[q]. With the bias
// Y = X + 0x808080808080 the lower six balanced digits are the bytes of Y XOR 0x80 (sigma + 128 is the
// plain base-256 digit of Y) and the top digit is byte 6 of Y (|sigma_0| <= 65), so digit s is byte
// 6 - s of Z = Y ^ 0x808080808080; byte gathers by PRMT.
__device__ __forceinline__ void oz_digits4(const double (&v)[4], int ex, double sc, uint32_t (&w)[OZ_S]) {
  uint32_t lo[4], hi[4];
  const long long lim = (1LL << 54) - 1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    long long X = __double2ll_rn(sc != 0.0 ? v[q] * sc : ldexp(v[q], 54 - ex));
    X = X > lim ? lim : (X < -lim ? -lim : X);
    const unsigned long long Z = (unsigned long long)(X + 0x808080808080LL) ^ 0x808080808080ULL;
    lo[q] = (uint32_t)Z;
    hi[q] = (uint32_t)(Z >> 32);
  }
#pragma unroll
  for (int s = 0; s < OZ_S; ++s) {
    const int j = (6 - s) & 3;                 // byte within the 32-bit half
    const uint32_t* src = (6 - s) >= 4 ? hi : lo;
    const uint32_t sel = (uint32_t)j | ((uint32_t)(4 + j) << 4);
    const uint32_t t01 = __byte_perm(src[0], src[1], sel), t23 = __byte_perm(src[2], src[3], sel);
    w[s] = __byte_perm(t01, t23, 0x5410);
  }
}

// row slices of a row-major (rows x K, ld) matrix into out[s][rows][K]: 4 consecutive k per thread
// (two 16-byte loads when aligned; a warp reads 1 KB contiguous), one 32-bit store per slice plane
__global__ void oz_slice_rows_kernel(int rows, int K, const double* __restrict__ X, long long ld,
                                     const int* __restrict__ e, uint8_t* out) {
  const int kq = K / 4;
  const long long plane = (long long)rows * K;
  const long long quads = (long long)rows * kq;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= quads) return;
  int r = (int)(g / kq), k = (int)(g - (long long)r * kq);
  const int dr = (int)(stride / kq), dk = (int)(stride - (long long)dr * kq);
  const bool al = ((reinterpret_cast<uintptr_t>(X) | (uintptr_t)(ld * 8)) & 15) == 0;
  for (; g < quads; g += stride) {
    const double* x = X + (long long)r * ld + 4 * k;
    double v[4];
    if (al) {
      const double2 a = __ldg(reinterpret_cast<const double2*>(x)), b = __ldg(reinterpret_cast<const double2*>(x) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldg(x + q);
    }
    const int ex = e[r];
    const double sc = oz_scale_of(ex);
    uint32_t w[OZ_S];
    oz_digits4(v, ex, sc, w);
    uint8_t* o = out + (long long)r * K + 4 * k;
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(o + s * plane) = w[s];
    k += dk;
    r += dr;
    if (k >= kq) { k -= kq; ++r; }
  }
}

// column slices of a row-major (K x cols, ld) matrix, transposed: out[s][cols][K]. 64 x 64 tiles: each
// thread digitizes 4 consecutive k of one column (coalesced row reads across the warp) into one word
// per plane, staged in shared memory [s][col][k/4] (17-word rows), then written as 64-byte K runs.
__global__ void __launch_bounds__(256) oz_slice_cols_kernel(int K, int cols, const double* __restrict__ X, long long ld,
                                                            const int* __restrict__ e, uint8_t* out) {
  __shared__ uint32_t t[OZ_S][64][17];
  const int k0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  const long long plane = (long long)cols * K;
  for (int it = threadIdx.x; it < 64 * 16; it += 256) {
    const int cc = it & 63, kq = it >> 6;
    const int c = c0 + cc;
    uint32_t w[OZ_S];
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) w[s] = 0;
    if (c < cols) {
      const int ex = e[c];
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + 4 * kq + q;
        v[q] = k < K ? __ldg(X + (long long)k * ld + c) : 0.0;
      }
      oz_digits4(v, ex, oz_scale_of(ex), w);
    }
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) t[s][cc][kq] = w[s];
  }
  __syncthreads();
  for (int it = threadIdx.x; it < OZ_S * 64 * 16; it += 256) {
    const int kq = it & 15, cc = (it >> 4) & 63, s = it >> 10;
    const int c = c0 + cc, k = k0 + 4 * kq;
    if (c < cols && k < K) *reinterpret_cast<uint32_t*>(out + s * plane + (long long)c * K + k) = t[s][cc][kq];
  }
}

PFN_cuTensorMapEncodeTiled_v12000 oz_encode() {
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

// slice stack [S][rows][K] int8, box box_k bytes x box_rows x S (32 / 64 / 128 bytes: matching swizzle)
bool oz_tmap(CUtensorMap* tm, const void* ptr, int rows, int K, int box_rows, int box_k) {
  auto enc = oz_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)OZ_S};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)rows * K};
  cuuint32_t box[3] = {(cuuint32_t)box_k, (cuuint32_t)box_rows, (cuuint32_t)OZ_S};
  cuuint32_t es[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = box_k == 32   ? CU_TENSOR_MAP_SWIZZLE_32B
                                : box_k == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                              : CU_TENSOR_MAP_SWIZZLE_128B;
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

namespace {
bool oz_shape_ok(int M, int N, int K) { return M > 0 && N > 0 && K > 0 && M % 128 == 0 && N % 64 == 0 && K % 64 == 0; }

int oz_nsm() {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  return nsm;
}

long long oz_tiles(int M, int N, int sym) {
  const long long ntn = N / OA_N, nmt = M / OZ_M;
  if (!sym) return nmt * ntn;
  long long t = 0;
  for (long long mt = 0; mt < nmt; ++mt) t += ntn - 2 * mt > 0 ? ntn - 2 * mt : 0;
  return t;
}

// K ranges: with fewer output tiles than SMs the K dimension is split (ranges >= 1024 deep) to fill
// the persistent grid; the split count maximizes units / (SMs x rounds), ties to fewer splits
void oz_split(long long tiles, int K, int* ks, int* kchunk) {
  const int nsm = oz_nsm();
  static const int long_kc = [] {
    const char* e = getenv("TTB_OZAKI_LONGK_CHUNK");
    return e ? atoi(e) : 4 * OZ_SUB * OA_K;
  }();
  if (K > 2 * long_kc && long_kc > 0 && tiles * ((K + long_kc - 1) / long_kc) >= 2LL * nsm) {
    // long K: 16384-deep ranges (4 TMEM accumulations), ordered range-major, so the CTAs running together all
    // read the same few thousand columns of the slice stacks (L2-resident) instead of drifting apart
    // over two halves of a multi-GB stack; costs ks partial tiles in HBM (reduced in a fixed order)
    *kchunk = (long_kc + OA_K - 1) / OA_K * OA_K;
    *ks = (K + *kchunk - 1) / *kchunk;
    return;
  }
  int best = 1;
  double best_eff = 0.0;
  const int kmax = K / 1024 > 1 ? K / 1024 : 1;
  for (int s = 1; s <= kmax && s <= 256; ++s) {
    const long long units = tiles * s;
    const long long rounds = (units + nsm - 1) / nsm;
    const double eff = (double)units / ((double)rounds * nsm);
    if (eff > best_eff * 1.02) { best_eff = eff; best = s; }
    if (tiles * s >= 4LL * nsm) break;
  }
  int kc = (int)(((long long)K + best - 1) / best);
  kc = (kc + OA_K - 1) / OA_K * OA_K;
  *kchunk = kc;
  *ks = (K + kc - 1) / kc;
}

struct OzWs {
  uint8_t *As, *Bs;
  int *ea, *fb;
  unsigned long long *amax, *bmax;
  double* part;
  long long bytes;
};

// gram: A and B are the same slice stack (B's pointers alias A's)
OzWs oz_ws_layout(void* base, int M, int N, int K, int gram) {
  int ks, kc;
  oz_split(oz_tiles(M, N, gram), K, &ks, &kc);
  OzWs w;
  uintptr_t p = reinterpret_cast<uintptr_t>(base);
  const uintptr_t p0 = p;
  auto take = [&](long long bytes) { const uintptr_t r = p; p = (p + bytes + 255) & ~uintptr_t(255); return r; };
  w.As = reinterpret_cast<uint8_t*>(take((long long)OZ_S * M * K));
  w.Bs = gram ? w.As : reinterpret_cast<uint8_t*>(take((long long)OZ_S * N * K));
  w.ea = reinterpret_cast<int*>(take(4LL * M));
  w.fb = gram ? w.ea : reinterpret_cast<int*>(take(4LL * N));
  w.amax = reinterpret_cast<unsigned long long*>(take(8LL * M));
  w.bmax = gram ? w.amax : reinterpret_cast<unsigned long long*>(take(8LL * N));
  w.part = reinterpret_cast<double*>(take(ks > 1 ? 8LL * ks * M * N : 8));
  w.bytes = (long long)(p - p0) + 256;
  return w;
}

// Row exponent + slicing in ONE pass (K % 4 == 0, K <= 128 NQ): one warp per row holds the row in
// registers (lane l: quads l + 32 j), takes the max, then writes the 7 slice planes -- the operand is
// read once instead of twice (oz_rowexp_kernel + oz_slice_rows_kernel: 8.6 GB of extra reads per
// 1M x 1024 operand).
template <int NQ>
__global__ void __launch_bounds__(256) oz_rowslice_fused_kernel(int rows, int K, const double* __restrict__ X,
                                                                 long long ld, int* __restrict__ e, uint8_t* out) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int kq = K / 4;
  const long long plane = (long long)rows * K;
  const double* x = X + (long long)r * ld;
  const bool al = ((reinterpret_cast<uintptr_t>(X) | (uintptr_t)(ld * 8)) & 15) == 0;
  double v[NQ][4];
  double m = 0.0;
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    const int q = lane + 32 * j;
    if (q < kq) {
      if (al) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(x + 4 * q));
        const double2 b = __ldg(reinterpret_cast<const double2*>(x + 4 * q) + 1);
        v[j][0] = a.x; v[j][1] = a.y; v[j][2] = b.x; v[j][3] = b.y;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) v[j][u] = __ldg(x + 4 * q + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) m = oz_amax(m, v[j][u]);
    }
  }
  for (int o = 16; o; o >>= 1) m = oz_amax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int ex = oz_exp_of(m);
  if (lane == 0) e[r] = ex;
  const double sc = oz_scale_of(ex);
  uint8_t* o = out + (long long)r * K;
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    const int q = lane + 32 * j;
    if (q < kq) {
      uint32_t w[OZ_S];
      oz_digits4(v[j], ex, sc, w);
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(o + s * plane + 4 * q) = w[s];
    }
  }
}

// The same with the rows staged in shared memory by 1-D bulk copies (cp.async.bulk, one per row of K * 8
// bytes, 16-byte aligned rows): 8 rows per CTA, <= 64 KB, so 3 CTAs per SM keep ~190 KB of loads in flight
// per SM with few registers, and the load / slice / store phases of different CTAs overlap. The register
// version (oz_rowslice_fused_kernel, 94 registers: 2 CTAs per SM) reached 3.6 TB/s on 1M x 1024.
template <int NQ>
__global__ void __launch_bounds__(256) oz_rowslice_bulk_kernel(int rows, int K, const double* __restrict__ X,
                                                                long long ld, int* __restrict__ e, uint8_t* out) {
  extern __shared__ __align__(128) double oz_rs[];
  __shared__ __align__(8) unsigned long long bar[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + w;
  if (r >= rows) return;
  const double* row = oz_rs + (size_t)w * K;
  const uint32_t mb = smem_u32(&bar[w]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(K * 8) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(row)),
                 "l"(X + (long long)r * ld), "r"(K * 8), "r"(mb)
                 : "memory");
  }
  __syncwarp();
  mbar_wait(mb, 0);
  const int kq = K / 4;
  const long long plane = (long long)rows * K;
  double m = 0.0;
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    const int q = lane + 32 * j;
    if (q < kq) {
      const double2 a = reinterpret_cast<const double2*>(row + 4 * q)[0];
      const double2 b = reinterpret_cast<const double2*>(row + 4 * q)[1];
      m = oz_amax(oz_amax(m, a.x), a.y);
      m = oz_amax(oz_amax(m, b.x), b.y);
    }
  }
  for (int o = 16; o; o >>= 1) m = oz_amax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int ex = oz_exp_of(m);
  if (lane == 0) e[r] = ex;
  const double sc = oz_scale_of(ex);
  uint8_t* o = out + (long long)r * K;
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    const int q = lane + 32 * j;
    if (q < kq) {
      const double2 a = reinterpret_cast<const double2*>(row + 4 * q)[0];
      const double2 b = reinterpret_cast<const double2*>(row + 4 * q)[1];
      const double v[4] = {a.x, a.y, b.x, b.y};
      uint32_t wd[OZ_S];
      oz_digits4(v, ex, sc, wd);
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(o + s * plane + 4 * q) = wd[s];
    }
  }
}

// Row exponent + slicing with zero padding to Mp x Kp (any K): one warp per row, max pass then slice pass
// (the second read of the row hits L1/L2); rows >= rows are zero with exponent 0.
__global__ void __launch_bounds__(256) oz_prows_kernel(int rows, int K, const double* __restrict__ X, long long ld,
                                                       int Mp, int Kp, int* __restrict__ e, uint8_t* out) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= Mp) return;
  const long long plane = (long long)Mp * Kp;
  uint8_t* o = out + (long long)r * Kp;
  if (r >= rows) {
    for (int q = lane; q < Kp / 4; q += 32)
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(o + s * plane + 4 * q) = 0u;
    if (lane == 0) e[r] = 0;
    return;
  }
  const double* x = X + (long long)r * ld;
  double m = 0.0;
  for (int k = lane; k < K; k += 32) m = oz_amax(m, __ldg(x + k));
  for (int of = 16; of; of >>= 1) m = oz_amax(m, __shfl_xor_sync(0xffffffffu, m, of));
  const int ex = oz_exp_of(m);
  if (lane == 0) e[r] = ex;
  const double sc = oz_scale_of(ex);
  for (int q = lane; q < Kp / 4; q += 32) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = 4 * q + u < K ? __ldg(x + 4 * q + u) : 0.0;
    uint32_t w[OZ_S];
    oz_digits4(v, ex, sc, w);
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint32_t*>(o + s * plane + 4 * q) = w[s];
  }
}

// TTB_OZ_BULK=0: the register-staged slicers (A/B comparison)
bool oz_bulk_rows() {
  static const bool on = getenv("TTB_OZ_BULK") == nullptr || getenv("TTB_OZ_BULK")[0] != '0';
  return on;
}

// exponents (and slices) of the rows of a row-major (rows x K, ld) operand
void oz_rows(cudaStream_t st, int rows, int K, const double* X, long long ld, int* e, unsigned long long* rmax,
             uint8_t* out) {
  if (K > 16384) {
    cudaMemsetAsync(rmax, 0, sizeof(unsigned long long) * rows, st);
    oz_rowmax_kernel<<<dim3(ceil_div(rows, 8), ceil_div(K, 8192)), 256, 0, st>>>(rows, K, X, ld, rmax); ttb_count();
    oz_colexp_kernel<<<ceil_div(rows, 256), 256, 0, st>>>(rows, rmax, e); ttb_count();
  } else if (K % 4 == 0 && K <= 128 * 8 && oz_bulk_rows() &&
             ((reinterpret_cast<uintptr_t>(X) | (uintptr_t)(ld * 8)) & 15) == 0) {
    const unsigned g = (unsigned)ceil_div((long long)rows, 8);
    const size_t sm = (size_t)8 * K * sizeof(double);
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(oz_rowslice_bulk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(oz_rowslice_bulk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cudaFuncSetAttribute(oz_rowslice_bulk_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cfg = true;
    }
    if (K <= 128 * 2) oz_rowslice_bulk_kernel<2><<<g, 256, sm, st>>>(rows, K, X, ld, e, out);
    else if (K <= 128 * 4) oz_rowslice_bulk_kernel<4><<<g, 256, sm, st>>>(rows, K, X, ld, e, out);
    else oz_rowslice_bulk_kernel<8><<<g, 256, sm, st>>>(rows, K, X, ld, e, out);
    ttb_count();
    return;
  } else if (K % 4 == 0 && K <= 128 * 16) {
    const unsigned g = (unsigned)ceil_div((long long)rows * 32, 256);
    if (K <= 128 * 2) oz_rowslice_fused_kernel<2><<<g, 256, 0, st>>>(rows, K, X, ld, e, out);
    else if (K <= 128 * 4) oz_rowslice_fused_kernel<4><<<g, 256, 0, st>>>(rows, K, X, ld, e, out);
    else if (K <= 128 * 8) oz_rowslice_fused_kernel<8><<<g, 256, 0, st>>>(rows, K, X, ld, e, out);
    else oz_rowslice_fused_kernel<16><<<g, 256, 0, st>>>(rows, K, X, ld, e, out);
    ttb_count();
    return;
  } else {
    oz_rowexp_kernel<<<ceil_div((long long)rows * 32, 256), 256, 0, st>>>(rows, K, X, ld, e); ttb_count();
  }
  oz_slice_rows_kernel<<<ttb_num_sms() * 16, 256, 0, st>>>(rows, K, X, ld, e, out); ttb_count();
}

// exponents (and transposed slices) of the columns of a row-major (K x cols, ld) operand
// Column exponent + transposed slicing in one kernel for short K (K <= 2048): a CTA owns 64 columns
// over all K rows -- pass 1 takes the column maxima (DRAM), pass 2 re-reads the CTA's 64 x K tile
// (<= 1 MB, L2-resident across the ~148 concurrent CTAs) and slices through the shared-memory
// transpose of oz_slice_cols_kernel. Saves the separate oz_colmax pass over the operand from DRAM.
__global__ void __launch_bounds__(256) oz_cols_fused_kernel(int K, int cols, const double* __restrict__ X, long long ld,
                                                            int* __restrict__ e, uint8_t* out) {
  __shared__ uint32_t t[OZ_S][64][17];
  __shared__ double pm[4][64];
  __shared__ int es[64];
  const int c0 = blockIdx.x * 64;
  const long long plane = (long long)cols * K;
  {
    const int cc = threadIdx.x & 63, kr = threadIdx.x >> 6;
    const int c = c0 + cc;
    double m = 0.0;
    if (c < cols)
      for (int k = kr; k < K; k += 4) m = oz_amax(m, __ldg(X + (long long)k * ld + c));
    pm[kr][cc] = m;
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const double m = oz_amax(oz_amax(pm[0][threadIdx.x], pm[1][threadIdx.x]), oz_amax(pm[2][threadIdx.x], pm[3][threadIdx.x]));
    const int ex = oz_exp_of(m);
    es[threadIdx.x] = ex;
    if (c0 + (int)threadIdx.x < cols) e[c0 + threadIdx.x] = ex;
  }
  __syncthreads();
  for (int k0 = 0; k0 < K; k0 += 64) {
    for (int it = threadIdx.x; it < 64 * 16; it += 256) {
      const int cc = it & 63, kq = it >> 6;
      const int c = c0 + cc;
      uint32_t w[OZ_S];
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) w[s] = 0;
      if (c < cols) {
        const int ex = es[cc];
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = k0 + 4 * kq + q;
          v[q] = k < K ? __ldg(X + (long long)k * ld + c) : 0.0;
        }
        oz_digits4(v, ex, oz_scale_of(ex), w);
      }
#pragma unroll
      for (int s = 0; s < OZ_S; ++s) t[s][cc][kq] = w[s];
    }
    __syncthreads();
    for (int it = threadIdx.x; it < OZ_S * 64 * 16; it += 256) {
      const int kq = it & 15, cc = (it >> 4) & 63, s = it >> 10;
      const int c = c0 + cc, k = k0 + 4 * kq;
      if (c < cols && k < K) *reinterpret_cast<uint32_t*>(out + s * plane + (long long)c * K + k) = t[s][cc][kq];
    }
    __syncthreads();
  }
}

// Column exponent + transposed slicing with the CTA's 8 columns x K rows (64-byte row segments, <= 64 KB)
// staged in shared memory by 16-byte cp.async: the operand is read from DRAM exactly once (the two-pass
// oz_cols_fused_kernel re-reads its tile and, with ~5 CTAs x 512 KB per SM in flight, misses L2: 17.2 GB
// read for an 8.6 GB operand). Row k sits at smem row k ^ ((k >> 4) & 1) so that the slice pass (thread =
// one column x 16 consecutive k; a warp covers 4 such k-groups 16 rows apart) reads conflict-free; it
// writes 16 bytes per slice plane (out[s][c][k], K contiguous).
__global__ void __launch_bounds__(256) oz_cols_stage_kernel(int K, int cols, const double* __restrict__ X, long long ld,
                                                            int* __restrict__ e, uint8_t* out) {
  extern __shared__ __align__(128) double oz_cs[];   // [K][8]
  __shared__ double pm[8][4][2];
  __shared__ int es[8];
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
  const int c0 = blockIdx.x * 8;
  const long long plane = (long long)cols * K;
  for (int idx = t; idx < 4 * K; idx += 256) {
    const int k = idx >> 2, ch = idx & 3;
    const int ks = k ^ ((k >> 4) & 1);
    const uint32_t dst = smem_u32(oz_cs + ks * 8 + 2 * ch);
    const double* src = X + (long long)k * ld + c0 + 2 * ch;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  {
    // column maxima: thread t always sees 16-byte chunk t & 3 (columns 2 (t & 3), 2 (t & 3) + 1)
    double m0 = 0.0, m1 = 0.0;
    for (int idx = t; idx < 4 * K; idx += 256) {
      const double2 v = reinterpret_cast<const double2*>(oz_cs)[idx];
      m0 = oz_amax(m0, v.x);
      m1 = oz_amax(m1, v.y);
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      m0 = oz_amax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
      m1 = oz_amax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    if (lane < 4) {
      pm[wp][lane][0] = m0;
      pm[wp][lane][1] = m1;
    }
  }
  __syncthreads();
  if (t < 8) {
    double m = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m = oz_amax(m, pm[w][t >> 1][t & 1]);
    const int ex = oz_exp_of(m);
    es[t] = ex;
    e[c0 + t] = ex;
  }
  __syncthreads();
  const int c = t & 7;
  const int ex = es[c];
  const double sc = oz_scale_of(ex);
  uint8_t* o = out + (long long)(c0 + c) * K;
  for (int kb = (t >> 3) * 16; kb < K; kb += 32 * 16) {
    uint32_t wd[4][OZ_S];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = kb + 4 * g + u;
        v[u] = oz_cs[(k ^ ((k >> 4) & 1)) * 8 + c];
      }
      oz_digits4(v, ex, sc, wd[g]);
    }
#pragma unroll
    for (int s2 = 0; s2 < OZ_S; ++s2)
      *reinterpret_cast<uint4*>(o + s2 * plane + kb) = make_uint4(wd[0][s2], wd[1][s2], wd[2][s2], wd[3][s2]);
  }
}

void oz_cols(cudaStream_t st, int K, int cols, const double* X, long long ld, int* e, unsigned long long* cmax,
             uint8_t* out) {
  if (K <= 1024 && K % 16 == 0 && cols % 8 == 0 && oz_bulk_rows() &&
      ((reinterpret_cast<uintptr_t>(X) | (uintptr_t)(ld * 8)) & 15) == 0) {
    static bool cfg = false;
    if (!cfg) {
      cudaFuncSetAttribute(oz_cols_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
      cfg = true;
    }
    oz_cols_stage_kernel<<<cols / 8, 256, (size_t)K * 64, st>>>(K, cols, X, ld, e, out); ttb_count();
    return;
  }
  if (K <= 2048) {
    oz_cols_fused_kernel<<<ceil_div(cols, 64), 256, 0, st>>>(K, cols, X, ld, e, out); ttb_count();
    return;
  }
  cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * cols, st);
  oz_colmax_kernel<<<dim3(ceil_div(cols, 256), ceil_div(K, 256)), 256, 0, st>>>(K, cols, X, ld, cmax); ttb_count();
  oz_colexp_kernel<<<ceil_div(cols, 256), 256, 0, st>>>(cols, cmax, e); ttb_count();
  oz_slice_cols_kernel<<<dim3(ceil_div(cols, 64), ceil_div(K, 64)), 256, 0, st>>>(K, cols, X, ld, e, out); ttb_count();
}

// G[i][j] = G[j][i] below the computed block triangle (j < 128 floor(i / 128))
__global__ void oz_mirror_kernel(int n, double* G, long long ldg) {
  const long long tot = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    if (j < (i / OZ_M) * OZ_M) G[(long long)i * ldg + j] = G[(long long)j * ldg + i];
  }
}

template <int LEV, bool LONGK>
int oz_launch_cluster(cudaStream_t st, int grid, size_t smem, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N,
                      int K, int kc, int ks, int tiles, int sym, const int* ea, const int* fb, const OzOut& o) {
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(oz_gemm_kernel<LEV, LONGK, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = true;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(320);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const OzBand nob{};
  const cudaError_t e = cudaLaunchKernelEx(&lc, oz_gemm_kernel<LEV, LONGK, false, 2>, ta, tb, M, N, K, kc, ks, tiles, sym,
                                           ea, fb, o, nob);
  return e == cudaSuccess ? 0 : (int)e;
}

// Optional per-launch timing of oz_gemm_kernel (ttb_ozaki_kernel_events): CUDA events on the launching
// stream right around the kernel, so a caller's roofline record can use the kernel's own duration inside a
// running step (the slicing passes before it and the reduce / mirror after it are outside the pair).
struct OzEvent {
  cudaEvent_t a, b;
  int M, N, K, kind;   // kind 0 general, 1 Gram (sym), 2 A lower-triangular, 3 B upper-triangular, 4 TT-matvec core
};
std::vector<OzEvent> g_oz_events;
bool g_oz_events_on = false;
struct OzEventScope {
  cudaStream_t st;
  OzEvent ev;
  bool on;
  OzEventScope(cudaStream_t s, int M, int N, int K, int kind) : st(s), on(g_oz_events_on) {
    if (!on) return;
    ev = OzEvent{nullptr, nullptr, M, N, K, kind};
    cudaEventCreate(&ev.a);
    cudaEventCreate(&ev.b);
    cudaEventRecord(ev.a, st);
  }
  void stop() {
    if (!on) return;
    cudaEventRecord(ev.b, st);
    g_oz_events.push_back(ev);
    on = false;
  }
};

// the int8 GEMM over prepared slices + split-K reduction (+ mirror for sym)
int oz_run(cudaStream_t st, const OzWs& w, int M, int N, int K, double alpha, double beta, double* C, long long ldc,
           int sym, int trilA = 0, int mv = 0, int nv = 0) {
  CUtensorMap ta, tb;
  if (!oz_tmap(&ta, w.As, M, K, OZ_M, OA_K) || !oz_tmap(&tb, w.Bs, N, K, OA_N, OA_K)) return TTB_EARG;
  const size_t smem = (size_t)OA_ST * OA_SBYTES + 8 * 32 * OA_EPAD * sizeof(double) + 1024;
  static bool cfg_all = false;
  if (!cfg_all) {
    cudaFuncSetAttribute(oz_gemm_kernel<7, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(oz_gemm_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(oz_gemm_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg_all = true;
  }
  static const int levels = [] {
    const char* e = getenv("TTB_OZAKI_LEVELS");
    return e && atoi(e) == 7 ? 7 : 8;
  }();
  const long long tiles = oz_tiles(M, N, sym);
  int ks, kc;
  oz_split(tiles, K, &ks, &kc);
  OzOut o;
  if (ks > 1)
    o = OzOut{w.part, N, (long long)M * N, 1.0, 0.0, 1, 0};
  else
    o = OzOut{C, ldc, 0, alpha, beta, (alpha == 1.0 && beta == 0.0) ? 0 : 2,
              trilA == 1 && M == K ? 1 : (trilA == 2 && N == K ? 2 : 0), mv, nv};
  // unit order: column block fastest shares the A row block among the CTAs running together and streams
  // every A row block once, but reads the B stack once per row block; when A's whole slice stack stays
  // in L2 (<= 32 MB) and B's does not, row block fastest reads B once instead (ncu, 1024 x 1M x 1024:
  // 60.2 GB read with column-fastest order = 8 row blocks x 7.5 GB of B slices)
  static const bool mfast_on = !(getenv("TTB_OZAKI_MFAST") && atoi(getenv("TTB_OZAKI_MFAST")) == 0);
  o.mfast = (mfast_on && !sym && o.trilA == 0 && M < N && (long long)OZ_S * M * K <= (32LL << 20) &&
             (long long)OZ_S * N * K > (32LL << 20)) ? 1 : 0;
  const long long units = tiles * ks;
  const int grid = units < oz_nsm() ? (int)units : oz_nsm();
  // 2-CTA clusters that multicast the A tiles (TTB_OZAKI_CLUSTER: 0 off, 1 Grams only (default), 2 all):
  // the Grams (both operands one slice stack, ~148 CTAs reading the same k-slabs) are shared-bandwidth
  // bound (profiles/README.md), multicast halves their A traffic: 18.5 -> 15.4 ms on 1024 x 1M
  static const int cluster_mode = getenv("TTB_OZAKI_CLUSTER") ? atoi(getenv("TTB_OZAKI_CLUSTER")) : 1;
  const bool cluster = levels == 8 && tiles % 2 == 0 && grid % 2 == 0 && (cluster_mode == 2 || (cluster_mode == 1 && sym));
  if (cluster) o.mfast = 0;   // a cluster's two CTAs take consecutive units that must share the A row block
  OzEventScope evs(st, M, N, K, sym ? 1 : (o.trilA == 1 ? 2 : (o.trilA == 2 ? 3 : 0)));
  if (cluster && kc > OZ_SUB * OA_K) {
    const int e = oz_launch_cluster<8, true>(st, grid, smem, ta, tb, M, N, K, kc, ks, (int)tiles, sym, w.ea, w.fb, o);
    if (e) return e;
  } else if (cluster) {
    const int e = oz_launch_cluster<8, false>(st, grid, smem, ta, tb, M, N, K, kc, ks, (int)tiles, sym, w.ea, w.fb, o);
    if (e) return e;
  } else if (kc > OZ_SUB * OA_K)
    oz_gemm_kernel<8, true><<<grid, 320, smem, st>>>(ta, tb, M, N, K, kc, ks, (int)tiles, sym, w.ea, w.fb, o);
  else if (levels == 7)
    oz_gemm_kernel<7, false><<<grid, 320, smem, st>>>(ta, tb, M, N, K, kc, ks, (int)tiles, sym, w.ea, w.fb, o);
  else
    oz_gemm_kernel<8, false><<<grid, 320, smem, st>>>(ta, tb, M, N, K, kc, ks, (int)tiles, sym, w.ea, w.fb, o);
  evs.stop();
  ttb_count();
  if (ks > 1) {
    const long long tot = (long long)M * N;
    int blocks = ceil_div(tot, 256);
    if (blocks > ttb_num_sms() * 8) blocks = ttb_num_sms() * 8;
    oz_reduce_kernel<<<blocks, 256, 0, st>>>(mv > 0 ? mv : M, mv > 0 ? nv : N, ks, w.part, alpha, beta, C, ldc, M, N);
    ttb_count();
  }
  if (sym) {
    const long long tot = (long long)M * N;
    int blocks = ceil_div(tot, 256);
    if (blocks > ttb_num_sms() * 8) blocks = ttb_num_sms() * 8;
    oz_mirror_kernel<<<blocks, 256, 0, st>>>(M, C, ldc); ttb_count();
  }
  return ttb_last_error();
}
}  // namespace

// Workspace (bytes) of ttb_dgemm_ozaki: slice stacks of A and B, exponents, maxima, split-K partials.
static inline int oz_rup(int v, int m) { return (v + m - 1) / m * m; }
// any shape: the padded shape's workspace (Mp = M rounded up to 128, Np, Kp to 64)
long long ozaki_ws_bytes(int M, int N, int K) {
  if (M < 1 || N < 1 || K < 1) return 0;
  return oz_ws_layout(nullptr, oz_rup(M, OZ_M), oz_rup(N, OA_N), oz_rup(K, OA_K), 0).bytes;
}
int ozaki_gemm_padded(cudaStream_t st, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      const double* B, long long ldb, double beta, double* C, long long ldc, void* ws);
bool ozaki_shape_ok(int M, int N, int K) { return oz_shape_ok(M, N, K); }

// C (M x N, ldc) = alpha A B + beta C, FP64 via the Ozaki scheme on the INT8 tensor cores. A: row-major
// M x K (lda); B: row-major K x N (ldb) when tB == 0, N x K (ldb) when tB == 1. ws: ozaki_ws_bytes.
int ozaki_gemm(cudaStream_t st, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
               const double* B, long long ldb, double beta, double* C, long long ldc, void* ws) {
  if (M < 1 || N < 1 || K < 1) return TTB_EARG;
  if (!oz_shape_ok(M, N, K)) return ozaki_gemm_padded(st, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws);
  OzWs w = oz_ws_layout(ws, M, N, K, 0);
  oz_rows(st, M, K, A, lda, w.ea, w.amax, w.As);
  if (tB)
    oz_rows(st, N, K, B, ldb, w.fb, w.bmax, w.Bs);
  else
    oz_cols(st, K, N, B, ldb, w.fb, w.bmax, w.Bs);
  return oz_run(st, w, M, N, K, alpha, beta, C, ldc, 0);
}

// ---- banded batched FP64 product on the int8 tensor cores (the AMEn band contraction)
//   out[i, x, o] = sum_{t < 2h+1, r < Rin} Tp[i + t, r, x] Mt[i, t, r, o],   i < n
// (tensor_train/banded.py band_gemm, the ttb_band_gemm DMMA batch). Batch i is an X x K (K = (2h+1) Rin)
// by K x Rout product whose A operand is the K window of Tp blocks i .. i+2h, so the Tp blocks are shared
// by 2h+1 consecutive batches. A is sliced once per GROUP of G batches (blocks gG .. gG+G+2h-1, one
// exponent per row x over the group, i.e. 2^-54 relative to the row's maximum over G+2h consecutive mode
// indices instead of the batch's own 2h+1), each batch's A tiles are TMA boxes at K offset (i - gG) Rin of
// its group's stack; B (Mt[i]) is sliced per batch with per-column exponents. Padding: rows X -> Mp (128),
// columns Rout -> Np (64), K -> Kp (64); padded slices are zero. The kernel is oz_gemm_kernel<8, false,
// true> (same MMA schedule, level folding and epilogue; rows >= X and columns >= Rout are not written).
namespace {
// cmax[b Cp + c] = max_k |X[(b rs + k) ld + c]| over k < Kv with b rs + k < lim (sticky NaN as oz_amax)
__global__ void oz_bcolmax_kernel(int Kv, int Cv, int Cp, const double* __restrict__ X, long long ld, long long rs,
                                  long long lim, unsigned long long* cmax) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.z;
  if (c >= Cv) return;
  const int k0 = blockIdx.y * 256;
  const int k1 = (int)min((long long)min(Kv, k0 + 256), lim - (long long)b * rs);
  double m = 0.0;
  for (int k = k0; k < k1; ++k) m = oz_amax(m, X[((long long)b * rs + k) * ld + c]);
  atomicMax(cmax + (long long)b * Cp + c, (unsigned long long)__double_as_longlong(m));
}
__global__ void oz_bexp_kernel(long long total, const unsigned long long* cmax, int* e) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < total) e[i] = oz_exp_of(__longlong_as_double((long long)cmax[i]));
}
// out[((b 7 + s) Cp + c) Kp + k] = slice s of X[(b rs + k) ld + c] (transposed, zero-padded to Cp x Kp)
// K is laid out in blocks of Rp >= Rin (zero rows r >= Rin): output k = blk Rp + r <- source row blk Rin + r,
// so that every batch window starts at a multiple of the 64-byte TMA k step
__global__ void __launch_bounds__(256) oz_bslice_kernel(int Kv, int Cv, int Cp, int Kp, const double* __restrict__ X,
                                                        long long ld, long long rs, long long lim, int Rin, int Rp,
                                                        const int* __restrict__ e, uint8_t* out) {
  __shared__ uint32_t t[OZ_S][64][17];
  const int k0 = blockIdx.y * 64, c0 = blockIdx.x * 64, b = blockIdx.z;
  const long long plane = (long long)Cp * Kp;
  uint8_t* ob = out + (long long)b * OZ_S * plane;
  const long long kl = min((long long)Kv, lim - (long long)b * rs);
  for (int it = threadIdx.x; it < 64 * 16; it += 256) {
    const int cc = it & 63, kq = it >> 6;
    const int c = c0 + cc;
    uint32_t w[OZ_S];
#pragma unroll
    for (int q = 0; q < OZ_S; ++q) w[q] = 0;
    if (c < Cv) {
      const int ex = e[(long long)b * Cp + c];
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + 4 * kq + q;
        const int r = k % Rp, src = (k / Rp) * Rin + r;
        v[q] = (r < Rin && src < kl) ? __ldg(X + ((long long)b * rs + src) * ld + c) : 0.0;
      }
      oz_digits4(v, ex, oz_scale_of(ex), w);
    }
#pragma unroll
    for (int q = 0; q < OZ_S; ++q) t[q][cc][kq] = w[q];
  }
  __syncthreads();
  for (int it = threadIdx.x; it < OZ_S * 64 * 16; it += 256) {
    const int kq = it & 15, cc = (it >> 4) & 63, q = it >> 10;
    const int c = c0 + cc, k = k0 + 4 * kq;
    if (c < Cp && k < Kp) *reinterpret_cast<uint32_t*>(ob + q * plane + (long long)c * Kp + k) = t[q][cc][kq];
  }
}

void oz_bslice(cudaStream_t st, int nb, int Kv, int Cv, int Cp, int Kp, const double* X, long long ld, long long rs,
               long long lim, int Rin, int Rp, unsigned long long* cmax, int* e, uint8_t* out) {
  cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * (size_t)nb * Cp, st);
  oz_bcolmax_kernel<<<dim3(ceil_div(Cv, 256), ceil_div(Kv, 256), nb), 256, 0, st>>>(Kv, Cv, Cp, X, ld, rs, lim, cmax);
  ttb_count();
  oz_bexp_kernel<<<ceil_div((long long)nb * Cp, 256), 256, 0, st>>>((long long)nb * Cp, cmax, e); ttb_count();
  oz_bslice_kernel<<<dim3(Cp / 64, Kp / 64, nb), 256, 0, st>>>(Kv, Cv, Cp, Kp, X, ld, rs, lim, Rin, Rp, e, out);
  ttb_count();
}

struct OzBandLayout {
  int Mp, Np, Rp, Kb, Kp, Kg, ng;
  uint8_t *As, *Bs;
  int *ea, *fb;
  unsigned long long *amax, *bmax;
  long long bytes;
};

OzBandLayout oz_band_layout(void* base, int n, int h, int Rin, int Rout, int X, int G) {
  OzBandLayout w;
  w.Mp = (X + OZ_M - 1) / OZ_M * OZ_M;
  w.Np = (Rout + OA_N - 1) / OA_N * OA_N;
  w.Rp = (Rin + OA_K - 1) / OA_K * OA_K;           // K block per Tp block / band offset (64-byte aligned)
  w.Kb = (2 * h + 1) * Rin;
  w.Kp = (2 * h + 1) * w.Rp;
  w.Kg = (G - 1) * w.Rp + w.Kp;
  w.ng = (n + G - 1) / G;
  uintptr_t p = reinterpret_cast<uintptr_t>(base);
  const uintptr_t p0 = p;
  auto take = [&](long long bytes) { const uintptr_t r = p; p = (p + bytes + 255) & ~uintptr_t(255); return r; };
  w.As = reinterpret_cast<uint8_t*>(take((long long)w.ng * OZ_S * w.Mp * w.Kg));
  w.Bs = reinterpret_cast<uint8_t*>(take((long long)n * OZ_S * w.Np * w.Kp));
  w.ea = reinterpret_cast<int*>(take(4LL * w.ng * w.Mp));
  w.fb = reinterpret_cast<int*>(take(4LL * n * w.Np));
  w.amax = reinterpret_cast<unsigned long long*>(take(8LL * w.ng * w.Mp));
  w.bmax = reinterpret_cast<unsigned long long*>(take(8LL * n * w.Np));
  w.bytes = (long long)(p - p0) + 256;
  return w;
}

bool oz_tmap3(CUtensorMap* tm, const void* ptr, int K, int rows, int planes, int box_rows) {
  auto enc = oz_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)rows * K};
  cuuint32_t box[3] = {(cuuint32_t)OA_K, (cuuint32_t)box_rows, (cuuint32_t)OZ_S};
  cuuint32_t es[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = OA_K == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B;
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

TTB_API long long ttb_band_gemm_ozaki_workspace(int n, int h, int Rin, int Rout, int X, int G) {
  if (n < 1 || h < 0 || Rin < 1 || Rout < 1 || X < 1 || G < 1) return 0;
  return oz_band_layout(nullptr, n, h, Rin, Rout, X, G).bytes;
}

// Tp: (n + 2h, Rin, X) row-major (h zero blocks per end, banded.py _padded); Mt: (n, 2h+1, Rin, Rout);
// out: (n, X, Rout). ws: ttb_band_gemm_ozaki_workspace bytes. G: batches per A slice group.
TTB_API int ttb_band_gemm_ozaki(void* stream, int n, int h, int Rin, int Rout, int X, const double* Tp,
                                const double* Mt, double* out, void* ws, int G) {
  if (n < 1 || h < 0 || Rin < 1 || Rout < 1 || X < 1 || G < 1 || !ws) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  OzBandLayout w = oz_band_layout(ws, n, h, Rin, Rout, X, G);
  if (w.Kp > OZ_SUB * OA_K) return TTB_EARG;     // one TMEM accumulation per tile (K <= 4096)
  // A: group g = rows k of Tp blocks gG .. gG + G + 2h - 1 (row-major (rows x X), ld X)
  oz_bslice(st, w.ng, (G + 2 * h) * Rin, X, w.Mp, w.Kg, Tp, X, (long long)G * Rin, (long long)(n + 2 * h) * Rin, Rin,
            w.Rp, w.amax, w.ea, w.As);
  // B: batch i = Mt[i] as ((2h+1) Rin x Rout), ld Rout
  oz_bslice(st, n, w.Kb, Rout, w.Np, w.Kp, Mt, Rout, (long long)w.Kb, (long long)n * w.Kb, Rin, w.Rp, w.bmax, w.fb,
            w.Bs);
  // both stacks are [batch][slice][rows][K]: 3-D maps with 7 planes per batch (z = 7 batch)
  CUtensorMap ta, tb;
  if (!oz_tmap3(&ta, w.As, w.Kg, w.Mp, w.ng * OZ_S, OZ_M) || !oz_tmap3(&tb, w.Bs, w.Kp, w.Np, n * OZ_S, OA_N))
    return TTB_EARG;
  const size_t smem = (size_t)OA_ST * OA_SBYTES + 8 * 32 * OA_EPAD * sizeof(double) + 1024;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(oz_gemm_kernel<8, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = true;
  }
  const int tiles = (w.Mp / OZ_M) * (w.Np / OA_N);
  const long long units = (long long)tiles * n;
  const int grid = units < oz_nsm() ? (int)units : oz_nsm();
  OzOut o{out, Rout, 0, 1.0, 0.0, 0, 0};
  OzBand bd{G, w.Rp, w.Mp, w.Np, w.Kp, X, Rout, n, (long long)X * Rout};
  // the n-tiles of one batch share its A window: 2-CTA clusters multicast it (TTB_BAND_CLUSTER=0 disables)
  static const bool bcl = getenv("TTB_BAND_CLUSTER") == nullptr || getenv("TTB_BAND_CLUSTER")[0] != '0';
  if (bcl && tiles % 2 == 0 && grid % 2 == 0) {
    static bool cfg2 = false;
    if (!cfg2) {
      cudaFuncSetAttribute(oz_gemm_kernel<8, false, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cfg2 = true;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(320);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&lc, oz_gemm_kernel<8, false, true, 2>, ta, tb, w.Mp, w.Np, w.Kp, w.Kp, 1,
                                             tiles, 0, (const int*)w.ea, (const int*)w.fb, o, bd);
    ttb_count();
    return e == cudaSuccess ? ttb_last_error() : (int)e;
  }
  oz_gemm_kernel<8, false, true><<<grid, 320, smem, st>>>(ta, tb, w.Mp, w.Np, w.Kp, w.Kp, 1, tiles, 0, w.ea, w.fb, o, bd);
  ttb_count();
  return ttb_last_error();
}

// Padded general product: operands sliced into Mp x Kp / Np x Kp stacks with zero padding (rows by
// oz_prows_kernel, columns of a K x N B by the batched column slicer with nb = 1), the kernel runs the
// padded shape and writes only the M x N block (OzOut.mv / nv; split-K partials are reduced over it).
int ozaki_gemm_padded(cudaStream_t st, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                      const double* B, long long ldb, double beta, double* C, long long ldc, void* ws) {
  const int Mp = oz_rup(M, OZ_M), Np = oz_rup(N, OA_N), Kp = oz_rup(K, OA_K);
  OzWs w = oz_ws_layout(ws, Mp, Np, Kp, 0);
  oz_prows_kernel<<<ceil_div((long long)Mp * 32, 256), 256, 0, st>>>(M, K, A, lda, Mp, Kp, w.ea, w.As); ttb_count();
  if (tB) {
    oz_prows_kernel<<<ceil_div((long long)Np * 32, 256), 256, 0, st>>>(N, K, B, ldb, Np, Kp, w.fb, w.Bs); ttb_count();
  } else {
    oz_bslice(st, 1, K, N, Np, Kp, B, ldb, 0, K, Kp, Kp, w.bmax, w.fb, w.Bs);
  }
  return oz_run(st, w, Mp, Np, Kp, alpha, beta, C, ldc, 0, 0, M, N);
}

// ---- TT-matvec core contraction without the two regrouping passes (tensor_train/core.py tt_matvec):
//   Y[(a, c), i, (b, d)] = sum_j M[a, i, j, b] G[c, j, d]
// is the GEMM (rows (a, i, b), K = j) x (K = j, columns (c, d)); both operands are sliced straight from
// their TT-core layout -- every (a, i) block of M and every c block of G is a K x Cb row-major matrix
// whose Cb columns are rows of the slice stack (block-column slicing, per-row exponents over j) -- and
// the epilogue writes Y in its core layout (OzOut mode 3). Replaces the 2.15 GB operand permute and
// the 8.6 GB output permute of the configs[4] step.
namespace {
__global__ void __launch_bounds__(256) oz_blkcols_kernel(int K, int Cb, const double* __restrict__ X, int* __restrict__ e,
                                                         uint8_t* out, long long plane) {
  __shared__ uint32_t t[OZ_S][64][17];
  __shared__ double pm[256];
  __shared__ int es[64];
  const long long blk = blockIdx.x;
  const double* Xb = X + blk * (long long)K * Cb;
  // pass 1: column maxima over K (thread (kr, c): rows kr, kr + 256 / Cb, ...)
  const int per = 256 / Cb;
  {
    const int c = threadIdx.x % Cb, kr = threadIdx.x / Cb;
    double m = 0.0;
    if (kr < per)
      for (int k = kr; k < K; k += per) m = oz_amax(m, __ldg(Xb + (long long)k * Cb + c));
    pm[threadIdx.x] = m;
  }
  __syncthreads();
  if (threadIdx.x < Cb) {
    double m = 0.0;
    for (int r = 0; r < per; ++r) m = oz_amax(m, pm[r * Cb + threadIdx.x]);
    const int ex = oz_exp_of(m);
    es[threadIdx.x] = ex;
    e[blk * Cb + threadIdx.x] = ex;
  }
  __syncthreads();
  // pass 2: 64-deep k tiles, transposed through shared memory into rows blk Cb + c of the stack
  for (int k0 = 0; k0 < K; k0 += 64) {
    for (int it = threadIdx.x; it < Cb * 16; it += 256) {
      const int cc = it % Cb, kq = it / Cb;
      const int ex = es[cc];
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + 4 * kq + q;
        v[q] = k < K ? __ldg(Xb + (long long)k * Cb + cc) : 0.0;
      }
      uint32_t w[OZ_S];
      oz_digits4(v, ex, oz_scale_of(ex), w);
#pragma unroll
      for (int q = 0; q < OZ_S; ++q) t[q][cc][kq] = w[q];
    }
    __syncthreads();
    for (int it = threadIdx.x; it < OZ_S * Cb * 16; it += 256) {
      const int kq = it & 15, cc = (it >> 4) % Cb, q = (it >> 4) / Cb;
      const int k = k0 + 4 * kq;
      if (k < K) *reinterpret_cast<uint32_t*>(out + q * plane + (blk * Cb + cc) * (long long)K + k) = t[q][cc][kq];
    }
    __syncthreads();
  }
}
}  // namespace

TTB_API long long ttb_matvec_core_ozaki_workspace(int Ra, int n, int m, int Rb, int rc, int rd) {
  const long long M = (long long)Ra * n * Rb, N = (long long)rc * rd;
  if (M > 0x7fffffffLL || N > 0x7fffffffLL) return 0;
  return ozaki_ws_bytes((int)M, (int)N, m);
}

// Y (Ra rc, n, Rb rd) = the TT-matvec core of M (Ra, n, m, Rb) and G (rc, m, rd). Shapes: Ra n Rb % 128,
// rc rd % 64, m % 64, rd % 16 == 0, Rb and rd <= 64 (TTB_EARG otherwise; the caller falls back).
TTB_API int ttb_matvec_core_ozaki(void* stream, int Ra, int n, int m, int Rb, int rc, int rd, const double* Mc,
                                  const double* Gc, double* Y, void* ws) {
  const long long Ml = (long long)Ra * n * Rb, Nl = (long long)rc * rd;
  if (Ml > 0x7fffffffLL || Nl > 0x7fffffffLL || Ml % OZ_M || Nl % OA_N || m % OA_K || rd % 16 || Rb > 64 || rd > 64 ||
      Rb < 1 || 256 % Rb || 256 % rd)
    return TTB_EARG;
  const int M = (int)Ml, N = (int)Nl;
  cudaStream_t st = as_stream(stream);
  OzWs w = oz_ws_layout(ws, M, N, m, 0);
  oz_blkcols_kernel<<<(unsigned)((long long)Ra * n), 256, 0, st>>>(m, Rb, Mc, w.ea, w.As, (long long)M * m); ttb_count();
  oz_blkcols_kernel<<<(unsigned)rc, 256, 0, st>>>(m, rd, Gc, w.fb, w.Bs, (long long)N * m); ttb_count();
  CUtensorMap ta, tb;
  if (!oz_tmap(&ta, w.As, M, m, OZ_M, OA_K) || !oz_tmap(&tb, w.Bs, N, m, OA_N, OA_K)) return TTB_EARG;
  const size_t smem = (size_t)OA_ST * OA_SBYTES + 8 * 32 * OA_EPAD * sizeof(double) + 1024;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(oz_gemm_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(oz_gemm_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = true;
  }
  const long long tiles = oz_tiles(M, N, 0);
  int ks, kc;
  oz_split(tiles, m, &ks, &kc);
  if (ks > 1) return TTB_EARG;   // the scatter epilogue writes final values: no split-K partials
  OzOut o{Y, 0, 0, 1.0, 0.0, 3, 0, 0, 0, n, Rb, rc, rd};
  const int grid = tiles < oz_nsm() ? (int)tiles : oz_nsm();
  OzEventScope evs(st, M, N, m, 4);
  if (kc > OZ_SUB * OA_K)
    oz_gemm_kernel<8, true><<<grid, 320, smem, st>>>(ta, tb, M, N, m, kc, 1, (int)tiles, 0, w.ea, w.fb, o);
  else
    oz_gemm_kernel<8, false><<<grid, 320, smem, st>>>(ta, tb, M, N, m, kc, 1, (int)tiles, 0, w.ea, w.fb, o);
  evs.stop();
  ttb_count();
  return ttb_last_error();
}

// Per-launch timing of oz_gemm_kernel. enable = 1: drop earlier records and time every launch from now on
// (two CUDA events per launch on its stream); enable = 0: stop. Returns the number of records held.
TTB_API int ttb_ozaki_kernel_events(int enable) {
  if (enable) {
    for (auto& e : g_oz_events) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    g_oz_events.clear();
  }
  g_oz_events_on = enable != 0;
  return (int)g_oz_events.size();
}
// Reads up to cap records in launch order (after synchronizing on each end event): ms[i] = kernel duration,
// shape[4 i ..] = M, N, K, kind (0 general, 1 Gram, 2 A lower-triangular, 3 B upper-triangular, 4 TT-matvec
// core). Returns the number written.
TTB_API int ttb_ozaki_kernel_events_read(int cap, double* ms, int* shape) {
  int n = 0;
  for (auto& e : g_oz_events) {
    if (n >= cap) break;
    float t = 0.f;
    cudaEventSynchronize(e.b);
    cudaEventElapsedTime(&t, e.a, e.b);
    ms[n] = (double)t;
    shape[4 * n] = e.M; shape[4 * n + 1] = e.N; shape[4 * n + 2] = e.K; shape[4 * n + 3] = e.kind;
    ++n;
  }
  return n;
}

TTB_API long long ttb_ozaki_workspace(int M, int N, int K) { return ozaki_ws_bytes(M, N, K); }

// Whether ttb_dgemm_ozaki runs this shape without padding (M % 128, N % 64, K % 64; any K: ranges of
// 4096 are accumulated exactly in TMEM and combined in int64). Other shapes run padded (zero slices,
// masked epilogue); the caller weighs the padding waste (linalg.gemm).
TTB_API int ttb_ozaki_applies(int M, int N, int K) { return oz_shape_ok(M, N, K) ? 1 : 0; }

// C (M x N, ldc) = A op(B), FP64 via the Ozaki scheme (see ozaki_gemm). ws: ttb_ozaki_workspace bytes.
// Returns TTB_EARG for shapes ttb_ozaki_applies rejects.
TTB_API int ttb_dgemm_ozaki(void* stream, int tB, int M, int N, int K, const double* A, long long lda,
                            const double* B, long long ldb, double* C, long long ldc, void* ws) {
  return ozaki_gemm(as_stream(stream), tB, M, N, K, 1.0, A, lda, B, ldb, 0.0, C, ldc, ws);
}

// C = A B with A (M x M, lda) lower triangular (its strict upper triangle must be zero): row block
// m0 of C only runs the k steps below m0 + 128 (half the work of a square product; Q = X R^-1 of
// the CholeskyQR passes). B: row-major M x N (ldb). ws: ttb_ozaki_workspace(M, N, M) bytes.
TTB_API int ttb_dgemm_ozaki_trilA(void* stream, int M, int N, const double* A, long long lda, const double* B,
                                  long long ldb, double* C, long long ldc, void* ws) {
  if (!oz_shape_ok(M, N, M)) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  OzWs w = oz_ws_layout(ws, M, N, M, 0);
  oz_rows(st, M, M, A, lda, w.ea, w.amax, w.As);
  oz_cols(st, M, N, B, ldb, w.fb, w.bmax, w.Bs);
  return oz_run(st, w, M, N, M, 1.0, 0.0, C, ldc, 0, 1);
}

// C = A B with B (N x N, ldb) upper triangular (its strict lower triangle must be zero): column block
// n0 of C only runs the k steps below n0 + 64 (~half the work; Q = X R^-1 of the rounding's certified
// full-rank cores, output row-major as the core layout wants it). A: row-major M x N (lda).
// ws: ttb_ozaki_workspace(M, N, N) bytes.
TTB_API int ttb_dgemm_ozaki_triuB(void* stream, int M, int N, const double* A, long long lda, const double* B,
                                  long long ldb, double* C, long long ldc, void* ws) {
  if (!oz_shape_ok(M, N, N)) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  OzWs w = oz_ws_layout(ws, M, N, N, 0);
  oz_rows(st, M, N, A, lda, w.ea, w.amax, w.As);
  oz_cols(st, N, N, B, ldb, w.fb, w.bmax, w.Bs);
  return oz_run(st, w, M, N, N, 1.0, 0.0, C, ldc, 0, 2);
}

// General form: C = alpha A op(B) + beta C.
TTB_API int ttb_dgemm_ozaki_ex(void* stream, int tB, int M, int N, int K, double alpha, const double* A, long long lda,
                               const double* B, long long ldb, double beta, double* C, long long ldc, void* ws) {
  return ozaki_gemm(as_stream(stream), tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, ws);
}

// Gram matrix G (n x n, ldg) = X^T X of a row-major m x n X (ldx), FP64 via the Ozaki scheme: X's
// columns are sliced once (they are both operands), only the output tiles touching the upper block
// triangle are computed, the rest is mirrored. n % 128 == 0, m % 64 == 0.
TTB_API long long ttb_ozaki_gram_workspace(int m, int n) {
  if (!oz_shape_ok(n, n, m) || n % OZ_M) return 0;
  return oz_ws_layout(nullptr, n, n, m, 1).bytes;
}
TTB_API int ttb_ozaki_gram(void* stream, int m, int n, const double* X, long long ldx, double* G, long long ldg, void* ws) {
  if (!oz_shape_ok(n, n, m) || n % OZ_M) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  OzWs w = oz_ws_layout(ws, n, n, m, 1);
  oz_cols(st, m, n, X, ldx, w.ea, w.amax, w.As);
  return oz_run(st, w, n, n, m, 1.0, 0.0, G, ldg, 1);
}

// Gram matrix of the ROWS, G (n x n) = T T^T of a row-major n x m T (ldt): rows sliced once (long rows:
// two-pass maxima), upper block triangle computed, mirrored. n % 128 == 0, m % 64 == 0.
TTB_API long long ttb_ozaki_gram_rows_workspace(int n, int m) { return ttb_ozaki_gram_workspace(m, n); }
TTB_API int ttb_ozaki_gram_rows(void* stream, int n, int m, const double* T, long long ldt, double* G, long long ldg,
                                void* ws) {
  if (!oz_shape_ok(n, n, m) || n % OZ_M) return TTB_EARG;
  cudaStream_t st = as_stream(stream);
  OzWs w = oz_ws_layout(ws, n, n, m, 1);
  oz_rows(st, n, m, T, ldt, w.ea, w.amax, w.As);
  return oz_run(st, w, n, n, m, 1.0, 0.0, G, ldg, 1);
}
