// Exact sub-key logits (step a1; reading Q9 of DESIGN.md):
//   s[l][c] = RN32( sum_k x[l][k] * sub[c][k] )      (Eq.Logits)
// the fp32 round-to-nearest-even of the EXACT dot product of the stored inputs,
// so that routing (steps a2-a3) is bit-exact and independent of accumulation
// order, batch composition and rank.
//
//  limb_split_kernel     one warp per row: x_row = X * 2^E with X an integer,
//                        |X| < 2^22, E the row's finest exponent; X written as
//                        three balanced base-256 int8 digits (limb-major
//                        [3][rows][d]).  A row whose exponents span > 22 bits is
//                        flagged (digits zero) and recomputed by exact_dd_kernel.
//  gemm_i8_exact_kernel  tcgen05 kind::i8 (s8 x s8 -> s32 in TMEM): for each
//                        K block, the 9 digit products X_p . W_q^T accumulate
//                        into 5 TMEM accumulators D_s (s = p + q); every partial
//                        sum is an exact int32 (|digit product| <= 2^14, d <= 2^16).
//                        Epilogue: S = sum_s D_s 2^(8s) in int64 (exact),
//                        __ll2float_rn (correctly rounded) * 2^(E_x + E_w) (exact).
//  exact_dd_kernel       fp64 double-double (TwoSum) dot product + correct RN32
//                        of the (hi, lo) pair: the F32-mode path and the fallback
//                        for flagged rows.  Exact whenever the running sums fit
//                        106 bits (always for bf16 rows).
#include <cstdlib>
#include <string>

#include "router.cuh"
#include "tcgen05.cuh"

namespace omni {
namespace {
using namespace tc;


constexpr int kMaxBits = 22;  // |X| < 2^22 => three balanced base-256 digits fit int8

// ---------------------------------------------------------------------------
// bf16 bits -> (integer significand M >= 0, exponent eb) with value = +-M * 2^eb
__device__ __forceinline__ void bf16_parts(uint32_t v, uint32_t& M, int& eb) {
  const uint32_t E = (v >> 7) & 0xFF, m = v & 0x7F;
  if (E == 0) {
    M = m;
    eb = -133;
  } else {
    M = m | 0x80;
    eb = (int)E - 134;
  }
}

__global__ void __launch_bounds__(256)
    limb_split_kernel(const uint16_t* __restrict__ in, int64_t rows, int d, int8_t* __restrict__ limbs,
                      int32_t* __restrict__ expo, int32_t* __restrict__ bad_list,
                      int32_t* __restrict__ bad_count) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t r = gw; r < rows; r += nw) {
    const uint16_t* row = in + r * d;
    int emin = 1 << 20, emax = -(1 << 20);
    for (int c = lane * 8; c < d; c += 256) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + c);
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t v = (w4[i >> 1] >> ((i & 1) * 16)) & 0xFFFF;
        uint32_t M;
        int eb;
        bf16_parts(v, M, eb);
        if (M) {
          emin = min(emin, eb + (int)(__ffs(M) - 1));
          emax = max(emax, eb + 31 - (int)__clz(M));
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
      emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    const bool zero_row = emax < emin;
    const bool ok = zero_row || (emax - emin) < kMaxBits;
    const int E = zero_row ? 0 : emin;
    if (lane == 0) {
      expo[r] = E;
      if (!ok) bad_list[atomicAdd(bad_count, 1)] = (int32_t)r;
    }
    int8_t* l0 = limbs + r * d;
    int8_t* l1 = l0 + rows * d;
    int8_t* l2 = l1 + rows * d;
    for (int c = lane * 8; c < d; c += 256) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + c);
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
      uint32_t p0[2] = {0, 0}, p1[2] = {0, 0}, p2[2] = {0, 0};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t v = (w4[i >> 1] >> ((i & 1) * 16)) & 0xFFFF;
        uint32_t M;
        int eb;
        bf16_parts(v, M, eb);
        int32_t X = 0;
        if (ok && M) {
          const int sh = eb - E;  // >= -ctz(M) (E is the finest exponent), < kMaxBits
          X = sh >= 0 ? (int32_t)(M << sh) : (int32_t)(M >> (-sh));
          if (v & 0x8000) X = -X;
        }
        const int32_t d0 = ((X + 128) & 255) - 128;
        const int32_t x1 = (X - d0) >> 8;
        const int32_t d1 = ((x1 + 128) & 255) - 128;
        const int32_t d2 = (x1 - d1) >> 8;
        p0[i >> 2] |= ((uint32_t)d0 & 0xFF) << ((i & 3) * 8);
        p1[i >> 2] |= ((uint32_t)d1 & 0xFF) << ((i & 3) * 8);
        p2[i >> 2] |= ((uint32_t)d2 & 0xFF) << ((i & 3) * 8);
      }
      *reinterpret_cast<uint2*>(l0 + c) = make_uint2(p0[0], p0[1]);
      *reinterpret_cast<uint2*>(l1 + c) = make_uint2(p1[0], p1[1]);
      *reinterpret_cast<uint2*>(l2 + c) = make_uint2(p2[0], p2[1]);
    }
  }
}

// ---------------------------------------------------------------------------
#ifndef OMNI_I8_BN
#define OMNI_I8_BN 96  // 5 x 96 = 480 of 512 TMEM columns; N = 64 tiles are shared-memory-read bound (0.90 vs 0.71 ms at C3a)
#endif
#ifndef OMNI_I8_STAGES
#define OMNI_I8_STAGES 2  // 2 x 84 KB of limb tiles
#endif
constexpr int IBM = 128, IBN = OMNI_I8_BN, IBK = 128 /*bytes = int8 elements*/, kIStages = OMNI_I8_STAGES;
constexpr int kIABytes = IBM * IBK;  // one limb
constexpr int kIBBytes = IBN * IBK;
constexpr int kIStageBytes = 3 * kIABytes + 3 * kIBBytes;  // 72 KB
constexpr int kISmemBytes = kIStages * kIStageBytes + 1024 + 256;
constexpr int kITmemCols = 512;  // 5 accumulators x IBN (<= 96) columns, rounded up to a power of two
// instruction descriptor, kind::i8: D = s32, A = B = s8, K-major, M = 128, N = 64
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(IBN >> 3) << 17) |
                              ((uint32_t)(IBM >> 4) << 24);

struct I8Args {
  int M, N, K;     // M tokens, N = h*R sub-key rows, K = d
  const int32_t* ex;  // [M]
  const int32_t* ew;  // [N]
  float* out;         // [M][N]
};

// CN > 1: a cluster of CN CTAs along N shares the A (token) limbs: CTA r loads rows
// [r*IBM/CN, (r+1)*IBM/CN) of each A limb and multicasts them to the whole cluster,
// so each CTA pulls 1/CN of the A bytes from L2; a stage is released when the MMAs of
// all CN CTAs are done with it (their commits arrive on every CTA's empty barrier).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

template <int CN>
__global__ void __launch_bounds__(256, 1)
    gemm_i8_exact_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         I8Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                // [stage][limb] 16 KB
  uint8_t* sB = smem + kIStages * 3 * kIABytes;      // [stage][limb] 8 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kIStages * kIStageBytes);
  uint64_t* empty = full + kIStages;
  uint64_t* tfull = empty + kIStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * IBM, n0 = blockIdx.x * IBN;
  const int num_kb = (args.K + IBK - 1) / IBK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kIStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CN);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kITmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CN > 1) cluster_sync_all();  // peers' barriers are initialised before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t crank = CN > 1 ? cluster_rank() : 0;
  constexpr uint16_t kMask = (uint16_t)((1u << CN) - 1u);

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: 3 A limbs + 3 B limbs per K block ----------------
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % kIStages;
      mbar_wait(&empty[s], ((kb / kIStages) & 1) ^ 1);
      mbar_expect_tx(&full[s], kIStageBytes);
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        if (CN > 1) {
          constexpr int rows = IBM / CN;
          tma_load_2d_mc(&tmA, &full[s], sA + (s * 3 + p) * kIABytes + crank * rows * IBK, kb * IBK,
                         p * args.M + m0 + (int)crank * rows, kMask);
        } else {
          tma_load_2d(&tmA, &full[s], sA + (s * 3 + p) * kIABytes, kb * IBK, p * args.M + m0);
        }
        tma_load_2d(&tmB, &full[s], sB + (s * 3 + p) * kIBBytes, kb * IBK, p * args.N + n0);
      }
    }
    if (CN > 1)  // drain: every peer's commits for every stage have arrived before exit
      for (int kb = num_kb; kb < num_kb + kIStages; ++kb)
        mbar_wait(&empty[kb % kIStages], ((kb / kIStages) & 1) ^ 1);
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: D_{p+q} += X_p . W_q^T ----------------
    for (int kb = 0; kb < num_kb; ++kb) {
      const int s = kb % kIStages;
      mbar_wait(&full[s], (kb / kIStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const uint32_t a0 = smem_u32(sA + (s * 3 + p) * kIABytes);
          const uint32_t b0 = smem_u32(sB + (s * 3 + q) * kIBBytes);
          const bool first_pair = (p == 0 || q == 2);  // first (p, q) with this p + q in loop order
#pragma unroll
          for (int k = 0; k < IBK / 32; ++k)
            umma_i8(tmem + (uint32_t)((p + q) * IBN), sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32),
                    kIdescI8, !(kb == 0 && k == 0 && first_pair));
        }
      if (CN > 1) umma_commit_mc(&empty[s], kMask);
      else umma_commit(&empty[s]);
    }
    umma_commit(tfull);
  } else if (warp >= 4) {
    // ---------------- epilogue: exact int64 combination, one rounding ----------------
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int qd = warp - 4;
    const int row = m0 + qd * 32 + lane;
    const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16);
    const bool row_ok = row < args.M;
    const int exr = row_ok ? args.ex[row] : 0;
#pragma unroll 1
    for (int c = 0; c < IBN / 16; ++c) {
      uint32_t D[5][16];
#pragma unroll
      for (int s = 0; s < 5; ++s) tmem_ld16(tbase + s * IBN + c * 16, D[s]);
      tmem_wait_ld();
      const int col0 = n0 + c * 16;
      if (!row_ok || col0 >= args.N) continue;
      float o[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t S = (int64_t)(int32_t)D[0][j] + ((int64_t)(int32_t)D[1][j] << 8) +
                          ((int64_t)(int32_t)D[2][j] << 16) + ((int64_t)(int32_t)D[3][j] << 24) +
                          ((int64_t)(int32_t)D[4][j] << 32);
        const int col = min(col0 + j, args.N - 1);
        o[j] = ldexpf(__ll2float_rn(S), exr + args.ew[col]);
      }
      float* dst = args.out + (size_t)row * args.N + col0;
      if (col0 + 16 <= args.N && (args.N % 4) == 0) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int i = 0; i < 4; ++i) d4[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
      } else {
        for (int j = 0; j < 16 && col0 + j < args.N; ++j) dst[j] = o[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CN > 1) cluster_sync_all();  // no CTA leaves while a peer may still signal or fill it
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kITmemCols));
  }
}

// Persistent variant (CN = 1, the default): one CTA per SM walks the (m, n) tiles, n
// fastest (consecutive CTAs share the token limbs in L2); the TMA producer keeps its stage
// ring running across tiles, so the next tile's first K blocks load while the epilogue
// drains TMEM; 8 epilogue warps (two per TMEM lane quarter, one column half each).  The
// 480-column accumulator set is single-buffered: the MMAs of tile i+1 start once the
// epilogue has read tile i's accumulators (tempty).
constexpr int kIEpiWarps = 8;
__global__ void __launch_bounds__(128 + 32 * kIEpiWarps, 1)
    gemm_i8_persist_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           I8Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kIStages * 3 * kIABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kIStages * kIStageBytes);
  uint64_t* empty = full + kIStages;
  uint64_t* tfull = empty + kIStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_kb = (args.K + IBK - 1) / IBK;
  const int n_nt = (args.N + IBN - 1) / IBN;
  const int n_tiles = n_nt * ((args.M + IBM - 1) / IBM);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kIStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kIEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kITmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: one stage ring across all tiles ----------------
    int g = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int m0 = (t / n_nt) * IBM, n0 = (t % n_nt) * IBN;
      for (int kb = 0; kb < num_kb; ++kb, ++g) {
        const int s = g % kIStages;
        mbar_wait(&empty[s], ((g / kIStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], kIStageBytes);
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          tma_load_2d(&tmA, &full[s], sA + (s * 3 + p) * kIABytes, kb * IBK, p * args.M + m0);
          tma_load_2d(&tmB, &full[s], sB + (s * 3 + p) * kIBBytes, kb * IBK, p * args.N + n0);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: D_{p+q} += X_p . W_q^T ----------------
    int g = 0, it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      mbar_wait(tempty, (it & 1) ^ 1);  // the epilogue has read the previous tile
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kb = 0; kb < num_kb; ++kb, ++g) {
        const int s = g % kIStages;
        mbar_wait(&full[s], (g / kIStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const uint32_t a0 = smem_u32(sA + (s * 3 + p) * kIABytes);
            const uint32_t b0 = smem_u32(sB + (s * 3 + q) * kIBBytes);
            const bool first_pair = (p == 0 || q == 2);
#pragma unroll
            for (int k = 0; k < IBK / 32; ++k)
              umma_i8(tmem + (uint32_t)((p + q) * IBN), sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32),
                      kIdescI8, !(kb == 0 && k == 0 && first_pair));
          }
        umma_commit(&empty[s]);
      }
      umma_commit(tfull);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: exact int64 combination, one rounding ----------------
    const int e = warp - 4, qd = e & 3, h = e >> 2;
    constexpr int kChunks = IBN / 16;
    const int c_lo = h * kChunks / 2, c_hi = (h + 1) * kChunks / 2;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int m0 = (t / n_nt) * IBM, n0 = (t % n_nt) * IBN;
      const int row = m0 + qd * 32 + lane;
      const bool row_ok = row < args.M;
      const int exr = row_ok ? args.ex[row] : 0;
      mbar_wait(tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16);
#pragma unroll 1
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t D[5][16];
#pragma unroll
        for (int s = 0; s < 5; ++s) tmem_ld16(tbase + s * IBN + c * 16, D[s]);
        tmem_wait_ld();
        if (c == c_hi - 1) {  // every accumulator column of this warp is in registers
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(tempty)) : "memory");
        }
        const int col0 = n0 + c * 16;
        if (!row_ok || col0 >= args.N) continue;
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t S = (int64_t)(int32_t)D[0][j] + ((int64_t)(int32_t)D[1][j] << 8) +
                            ((int64_t)(int32_t)D[2][j] << 16) + ((int64_t)(int32_t)D[3][j] << 24) +
                            ((int64_t)(int32_t)D[4][j] << 32);
          const int col = min(col0 + j, args.N - 1);
          o[j] = ldexpf(__ll2float_rn(S), exr + args.ew[col]);
        }
        float* dst = args.out + (size_t)row * args.N + col0;
        if (col0 + 16 <= args.N && (args.N % 4) == 0) {
          float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
          for (int i = 0; i < 4; ++i) d4[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (col0 + j < args.N) dst[j] = o[j];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kITmemCols));
  }
}

// ---------------------------------------------------------------------------
// N4 (the selection never materialises the full
// score matrix): the persistent exact-logit GEMM with the per-half top-k' taken in its
// epilogue.  Work units are (128-token block, half of a head): a CTA walks the unit's
// column tiles in order, so each epilogue thread (one token row, one 48-column half of every
// tile) sees its half's columns one after another and keeps their top kp half keys
// (value desc, index asc -- the selection's key) in a sorted register list, plus the running
// (max, sum exp) of the logsumexp; at the unit's end it writes kp keys (+ one float2)
// instead of the half's logits.  Tiles past the half's end are computed and masked (the B
// rows beyond it belong to the next half or are TMA zero fill).
// + the epilogue scratch: 256 threads x 48 floats after the barriers (which take < 256 bytes)
constexpr int kISmemTopk = kIStages * kIStageBytes + 1024 + 256 + 256 * (IBN / 2) * 4;
static_assert(kISmemTopk <= 227 * 1024, "fused i8 GEMM shared memory");
struct I8TopArgs {
  int kp, R, n_rows, n_cols, n_heads;
  uint64_t* cand;         // [M][2h][2][kp]
  float2* part;           // [M][2h][2] or null
  const int32_t* counts;  // counts[1] > 0: flagged sub-key rows -> the logits are written too
};
__device__ __forceinline__ uint64_t fused_half_key(float v, uint32_t i) {
  v = v + 0.0f;  // -0.0 -> +0.0: equal values compare equal (the selection's half_key)
  return ((uint64_t)ord32(v) << 32) | (uint64_t)(0xFFFFFFFFu - i);
}
template <int KP>
__global__ void __launch_bounds__(128 + 32 * kIEpiWarps, 1)
    gemm_i8_topk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        I8Args args, I8TopArgs ta) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kIStages * 3 * kIABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kIStages * kIStageBytes);
  uint64_t* empty = full + kIStages;
  uint64_t* tfull = empty + kIStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_kb = (args.K + IBK - 1) / IBK;
  const int G = 2 * ta.n_heads;  // halves per token
  const int n_units = ((args.M + IBM - 1) / IBM) * G;
  auto unit = [&](int u, int& m0, int& c0, int& len) {
    const int g = u % G;
    m0 = (u / G) * IBM;
    c0 = (g >> 1) * ta.R + ((g & 1) ? ta.n_rows : 0);
    len = (g & 1) ? ta.n_cols : ta.n_rows;
  };

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kIStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kIEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kITmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    int g = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int m0, c0, len;
      unit(u, m0, c0, len);
      for (int n0 = c0; n0 < c0 + len; n0 += IBN)
        for (int kb = 0; kb < num_kb; ++kb, ++g) {
          const int s = g % kIStages;
          mbar_wait(&empty[s], ((g / kIStages) & 1) ^ 1);
          mbar_expect_tx(&full[s], kIStageBytes);
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            tma_load_2d(&tmA, &full[s], sA + (s * 3 + p) * kIABytes, kb * IBK, p * args.M + m0);
            tma_load_2d(&tmB, &full[s], sB + (s * 3 + p) * kIBBytes, kb * IBK, p * args.N + n0);
          }
        }
    }
  } else if (warp == 1 && lane == 0) {
    int g = 0, it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int m0, c0, len;
      unit(u, m0, c0, len);
      for (int n0 = c0; n0 < c0 + len; n0 += IBN, ++it) {
        mbar_wait(tempty, (it & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < num_kb; ++kb, ++g) {
          const int s = g % kIStages;
          mbar_wait(&full[s], (g / kIStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const uint32_t a0 = smem_u32(sA + (s * 3 + p) * kIABytes);
              const uint32_t b0 = smem_u32(sB + (s * 3 + q) * kIBBytes);
              const bool first_pair = (p == 0 || q == 2);
#pragma unroll
              for (int k = 0; k < IBK / 32; ++k)
                umma_i8(tmem + (uint32_t)((p + q) * IBN), sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32),
                        kIdescI8, !(kb == 0 && k == 0 && first_pair));
            }
          umma_commit(&empty[s]);
        }
        umma_commit(tfull);
      }
    }
  } else if (warp >= 4) {
    // the tile's values go through a per-thread shared-memory scratch (48 floats, thread-
    // contiguous words): the accumulators are released right after the TMEM reads, and the
    // list updates run while the MMAs of the next tile proceed
    const int e = warp - 4, qd = e & 3, h = e >> 2;
    constexpr int kChunks = IBN / 16, kCols = IBN / 2;
    const int c_lo = h * kChunks / 2, c_hi = (h + 1) * kChunks / 2;
    const int et = threadIdx.x - 128;
    float* scr = reinterpret_cast<float*>(smem + kIStages * kIStageBytes + 256) + et;
    const bool wlog = ta.counts[1] > 0;
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int m0, c0, len;
      unit(u, m0, c0, len);
      const int row = m0 + qd * 32 + lane;
      const bool row_ok = row < args.M;
      const int exr = row_ok ? args.ex[row] : 0;
      uint64_t lst[KP];
#pragma unroll
      for (int i = 0; i < KP; ++i) lst[i] = 0ull;
      float mx = -INFINITY, se = 0.f;
      for (int n0 = c0; n0 < c0 + len; n0 += IBN, ++it) {
        mbar_wait(tfull, it & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16);
#pragma unroll 1
        for (int c = c_lo; c < c_hi; ++c) {
          uint32_t D[5][16];
#pragma unroll
          for (int s = 0; s < 5; ++s) tmem_ld16(tbase + s * IBN + c * 16, D[s]);
          tmem_wait_ld();
          if (c == c_hi - 1) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(tempty)) : "memory");
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int64_t S = (int64_t)(int32_t)D[0][j] + ((int64_t)(int32_t)D[1][j] << 8) +
                              ((int64_t)(int32_t)D[2][j] << 16) + ((int64_t)(int32_t)D[3][j] << 24) +
                              ((int64_t)(int32_t)D[4][j] << 32);
            const int col = min(n0 + c * 16 + j, args.N - 1);
            scr[((c - c_lo) * 16 + j) * 256] = ldexpf(__ll2float_rn(S), exr + args.ew[col]);
          }
        }
        const int col0 = n0 + c_lo * 16;
        const int nv = row_ok ? max(0, min(kCols, c0 + len - col0)) : 0;  // this thread's columns in the half
        if (wlog && nv > 0) {
          float* dst = args.out + (size_t)row * args.N + col0;
          for (int j = 0; j < nv; ++j) dst[j] = scr[j * 256];
        }
        if (ta.part && nv > 0) {
          float cm = mx;
          for (int j = 0; j < nv; ++j) cm = fmaxf(cm, scr[j * 256]);
          float add = 0.f;
          for (int j = 0; j < nv; ++j) add += __expf(scr[j * 256] - cm);
          se = (mx == -INFINITY ? 0.f : se * __expf(mx - cm)) + add;
          mx = cm;
        }
        // the columns above the list's current threshold, then one insertion round per
        // pending column: the warp runs max over its lanes of the insertions, not one
        // round per column in which any lane inserts
        uint64_t pend = 0;
        for (int j = 0; j < nv; ++j)
          if (fused_half_key(scr[j * 256], (uint32_t)(col0 + j - c0)) > lst[KP - 1]) pend |= 1ull << j;
        while (__any_sync(0xffffffffu, pend != 0)) {
          if (pend) {
            const int j = __ffsll((long long)pend) - 1;
            pend &= pend - 1;
            const uint64_t key = fused_half_key(scr[j * 256], (uint32_t)(col0 + j - c0));
            if (key > lst[KP - 1]) {
#pragma unroll
              for (int i = KP - 1; i > 0; --i) lst[i] = key > lst[i - 1] ? lst[i - 1] : (key > lst[i] ? key : lst[i]);
              lst[0] = key > lst[0] ? key : lst[0];
            }
          }
        }
      }
      if (row_ok) {
        const int g = u % G;
        uint64_t* dst = ta.cand + (((size_t)row * G + g) * 2 + h) * ta.kp;
#pragma unroll
        for (int i = 0; i < KP; ++i)
          if (i < ta.kp) dst[i] = lst[i];
        if (ta.part) ta.part[((size_t)row * G + g) * 2 + h] = make_float2(mx, se);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kITmemCols));
  }
}

// ---------------------------------------------------------------------------
// exact fp64 double-double dot + correct RN32
template <typename T>
__device__ __forceinline__ double to_d(T v);
template <>
__device__ __forceinline__ double to_d<__nv_bfloat16>(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
template <>
__device__ __forceinline__ double to_d<float>(float v) { return (double)v; }

// RN32 of the exact value hi + lo, where hi = RN64(hi + lo).
__device__ __forceinline__ float rn32_dd(double hi, double lo) {
  const float f = __double2float_rn(hi);
  if ((double)f == hi || isinf(f)) return f;
  // neighbours of hi in fp32
  const float g = (double)f < hi ? nextafterf(f, INFINITY) : nextafterf(f, -INFINITY);
  const double mid = 0.5 * ((double)f + (double)g);  // exact in fp64
  if (hi != mid) return f;  // |lo| <= ulp64(hi)/2 cannot cross a midpoint that differs from hi
  if (lo == 0.0) return f;  // exact tie: __double2float_rn already rounded to even
  return ((lo > 0.0) == ((double)g > hi)) ? g : f;
}

// grid-stride over work items; mode 0: all (token, 128-column block) items;
// mode 1: tokens in list; mode 2: columns in list, 128-token blocks.
template <typename T>
__global__ void __launch_bounds__(128)
    exact_dd_kernel(const T* __restrict__ x, const T* __restrict__ sub, int d, int NC, int L,
                    float* __restrict__ logits, int mode, const int32_t* __restrict__ list,
                    const int32_t* __restrict__ list_count) {
  __shared__ double xs[128][33];
  __shared__ double ws[32];
  if (mode == 2) {
    const int ncols = *list_count;
    const int ntb = (L + 127) / 128;
    for (int item = blockIdx.x; item < ncols * ntb; item += gridDim.x) {
      const int c = list[item / ntb];
      const int l0 = (item % ntb) * 128;
      const int l = l0 + threadIdx.x;
      double s = 0.0, e = 0.0;
      for (int k0 = 0; k0 < d; k0 += 32) {
        __syncthreads();
        if (threadIdx.x < 32) ws[threadIdx.x] = (k0 + threadIdx.x < d) ? to_d(sub[(size_t)c * d + k0 + threadIdx.x]) : 0.0;
        for (int i = threadIdx.x; i < 128 * 32; i += 128) {
          const int rr = i / 32, kk = i % 32;
          xs[rr][kk] = (l0 + rr < L && k0 + kk < d) ? to_d(x[(size_t)(l0 + rr) * d + k0 + kk]) : 0.0;
        }
        __syncthreads();
        const int kmax = min(32, d - k0);
        for (int kk = 0; kk < kmax; ++kk) {
          const double p = xs[threadIdx.x][kk] * ws[kk];  // exact for bf16 / fp32 inputs
          const double t = s + p, bb = t - s;
          e += (s - (t - bb)) + (p - bb);
          s = t;
        }
      }
      if (l < L) {
        const double hi = s + e;
        logits[(size_t)l * NC + c] = rn32_dd(hi, e - (hi - s));
      }
    }
    return;
  }
  const int ncb = (NC + 127) / 128;
  const int nrows = mode == 1 ? *list_count : L;
  for (int item = blockIdx.x; item < nrows * ncb; item += gridDim.x) {
    const int l = mode == 1 ? list[item / ncb] : item / ncb;
    const int c0 = (item % ncb) * 128;
    const int c = c0 + threadIdx.x;
    double s = 0.0, e = 0.0;
    for (int k0 = 0; k0 < d; k0 += 32) {
      __syncthreads();
      if (threadIdx.x < 32) ws[threadIdx.x] = (k0 + threadIdx.x < d) ? to_d(x[(size_t)l * d + k0 + threadIdx.x]) : 0.0;
      for (int i = threadIdx.x; i < 128 * 32; i += 128) {
        const int rr = i / 32, kk = i % 32;
        xs[rr][kk] = (c0 + rr < NC && k0 + kk < d) ? to_d(sub[(size_t)(c0 + rr) * d + k0 + kk]) : 0.0;
      }
      __syncthreads();
      const int kmax = min(32, d - k0);
      for (int kk = 0; kk < kmax; ++kk) {
        const double p = ws[kk] * xs[threadIdx.x][kk];
        const double t = s + p, bb = t - s;
        e += (s - (t - bb)) + (p - bb);
        s = t;
      }
    }
    if (c < NC) {
      const double hi = s + e;
      logits[(size_t)l * NC + c] = rn32_dd(hi, e - (hi - s));
    }
  }
}

struct ExactWs {
  int8_t* limbs_x;
  int8_t* limbs_w;
  int32_t* ex;
  int32_t* ew;
  int32_t* bad_x;
  int32_t* bad_w;
  int32_t* counts;  // [2]: bad x rows, bad sub-key rows
};

size_t carve_exact(const omnimoe_dims& d, int64_t L, void* ws, ExactWs* o) {
  Carver c(ws);
  const int64_t NC = d.n_heads * (d.n_rows + d.n_cols);
  ExactWs w;
  w.limbs_x = c.take<int8_t>((size_t)3 * L * d.d);
  w.limbs_w = c.take<int8_t>((size_t)3 * NC * d.d);
  w.ex = c.take<int32_t>(std::max<int64_t>(L, 1));
  w.ew = c.take<int32_t>(NC);
  w.bad_x = c.take<int32_t>(std::max<int64_t>(L, 1));
  w.bad_w = c.take<int32_t>(NC);
  w.counts = c.take<int32_t>(2);
  if (o) *o = w;
  return c.bytes();
}

}  // namespace

size_t exact_logits_ws_bytes(const omnimoe_dims& d, int64_t L) {
  if (d.dtype != OMNIMOE_BF16) return 256;
  return carve_exact(d, L, nullptr, nullptr);
}

omnimoe_status launch_exact_dd(int dtype, const void* x, const void* sub, int d, int NC, int L,
                               float* logits, int mode, const int32_t* list, const int32_t* list_count,
                               cudaStream_t st) {
  int grid;
  if (mode == 0) grid = (int)std::min<int64_t>((int64_t)L * ((NC + 127) / 128), 1 << 30);
  else grid = num_sms() * 8;
  if (grid <= 0) return OMNIMOE_OK;
  if (dtype == OMNIMOE_BF16)
    exact_dd_kernel<__nv_bfloat16><<<grid, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(x),
                                                         static_cast<const __nv_bfloat16*>(sub), d, NC,
                                                         L, logits, mode, list, list_count);
  else
    exact_dd_kernel<float><<<grid, 128, 0, st>>>(static_cast<const float*>(x), static_cast<const float*>(sub),
                                                 d, NC, L, logits, mode, list, list_count);
  OMNI_CHECK_LAUNCH("exact_dd_kernel");
  return OMNIMOE_OK;
}

// K-only part of the rule (the workspace size must not depend on the device's SM count)
static int fused_kp_dims(const omnimoe_dims& d) {
  if (d.dtype != OMNIMOE_BF16 || d.router != OMNIMOE_ROUTER_EXACT || d.d >= 65536) return 0;
  const int64_t K1 = d.top_k + 1;
  if (K1 > 32 || K1 < 9) return 0;
  const int64_t kr1 = std::min<int64_t>(K1, d.n_rows), kc1 = std::min<int64_t>(K1, d.n_cols);
  int64_t C = 0;
  for (int64_t a = 1; a <= kr1; ++a) C += std::min<int64_t>(kc1, K1 / a);
  return C <= 160 ? (int)K1 : 0;
}
int fused_kp(const omnimoe_dims& d, int64_t L) {
  // small K only: the per-half lists (K+1 keys) are what the warp selection kernel takes
  // (launch_select: K+1 <= 32 and <= 160 product candidates); at large K a 48-column
  // segment would keep all its keys.  And only where it pays (the C2
  // sweep, profiles/r2/n4/): K >= 8 (below, the selection it saves is cheaper than the
  // list updates) and at least ~2/3 of the SMs' worth of (128-token block, half) units
  const int kp = fused_kp_dims(d);
  if (!kp || tuning().i8_cluster > 1 || !tuning().i8_persist || !tuning().route_fused) return 0;
  if (((L + IBM - 1) / IBM) * 2 * d.n_heads * 3 < 2 * (int64_t)num_sms()) return 0;
  return kp;
}
size_t fused_route_bytes(const omnimoe_dims& d, int64_t L) {
  const int kp = fused_kp_dims(d);  // reserved whenever K qualifies, whatever the device
  if (!kp) return 0;
  Carver c(nullptr);
  c.take<uint64_t>((size_t)std::max<int64_t>(L, 1) * 2 * d.n_heads * 2 * kp);
  c.take<float2>((size_t)std::max<int64_t>(L, 1) * 2 * d.n_heads * 2);
  return c.bytes();
}

omnimoe_status exact_logits(const omnimoe_dims& d, int64_t L, const void* x, const void* sub, float* logits,
                            void* ws, cudaStream_t st) {
  return exact_logits_fused(d, L, x, sub, logits, ws, nullptr, false, nullptr, st);
}

omnimoe_status exact_logits_fused(const omnimoe_dims& d, int64_t L, const void* x, const void* sub, float* logits,
                                  void* ws, void* fused_ws, bool want_part, FusedRoute* fr, cudaStream_t st) {
  const int NC = (int)(d.n_heads * (d.n_rows + d.n_cols));
  if (d.dtype != OMNIMOE_BF16)
    return launch_exact_dd(d.dtype, x, sub, (int)d.d, NC, (int)L, logits, 0, nullptr, nullptr, st);
  ExactWs w;
  carve_exact(d, L, ws, &w);
  if (cudaMemsetAsync(w.counts, 0, 2 * sizeof(int32_t), st) != cudaSuccess) {
    set_error("route: memset failed");
    return OMNIMOE_ERR_CUDA;
  }
  const int grid_x = (int)std::min<int64_t>((L + 7) / 8, num_sms() * 16);
  limb_split_kernel<<<std::max(grid_x, 1), 256, 0, st>>>(static_cast<const uint16_t*>(x), L, (int)d.d, w.limbs_x,
                                                         w.ex, w.bad_x, w.counts);
  OMNI_CHECK_LAUNCH("limb_split_kernel(x)");
  limb_split_kernel<<<(NC + 7) / 8, 256, 0, st>>>(static_cast<const uint16_t*>(sub), NC, (int)d.d, w.limbs_w,
                                                  w.ew, w.bad_w, w.counts + 1);
  OMNI_CHECK_LAUNCH("limb_split_kernel(subkeys)");

  for (auto k : {gemm_i8_exact_kernel<1>, gemm_i8_exact_kernel<2>, gemm_i8_exact_kernel<4>, gemm_i8_persist_kernel})
    if (!set_smem_attr(reinterpret_cast<const void*>(k), kISmemBytes)) {
      set_error("route: cannot set dynamic shared memory size of the i8 GEMM");
      return OMNIMOE_ERR_CUDA;
    }
  // clusters of CN CTAs along N multicast the A limbs (CN | number of N tiles)
  const int n_tiles = (NC + IBN - 1) / IBN;
  int CN = std::max(1, std::min(4, tuning().i8_cluster));
  while (CN > 1 && n_tiles % CN) CN >>= 1;
  CUtensorMap mA, mB;
  const bool ok =
      make_map_2d(&mA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, w.limbs_x, 3 * (uint64_t)L, d.d, IBK, IBM / CN) &&
      make_map_2d(&mB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, w.limbs_w, 3 * (uint64_t)NC, d.d, IBK, IBN);
  if (!ok) {
    set_error("route: cuTensorMapEncodeTiled failed for the limb operands");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  I8Args a{(int)L, NC, (int)d.d, w.ex, w.ew, logits};
  dim3 grid(n_tiles, (unsigned)((L + IBM - 1) / IBM));
  const int kp = fused_ws ? fused_kp(d, L) : 0;
  if (kp && CN == 1) {
    Carver c(fused_ws);
    I8TopArgs ta;
    ta.kp = kp;
    ta.R = (int)(d.n_rows + d.n_cols);
    ta.n_rows = (int)d.n_rows;
    ta.n_cols = (int)d.n_cols;
    ta.n_heads = (int)d.n_heads;
    ta.cand = c.take<uint64_t>((size_t)std::max<int64_t>(L, 1) * 2 * d.n_heads * 2 * kp);
    float2* part = c.take<float2>((size_t)std::max<int64_t>(L, 1) * 2 * d.n_heads * 2);
    ta.part = want_part ? part : nullptr;
    ta.counts = w.counts;
    const int64_t units = ((L + IBM - 1) / IBM) * 2 * d.n_heads;
    const int g = (int)std::min<int64_t>(units, num_sms());
    // list length = kp for the common K = 16 (kp = 17), else the next multiple of 8
    auto k = kp <= 8 ? gemm_i8_topk_kernel<8> : kp <= 16 ? gemm_i8_topk_kernel<16> : kp == 17 ? gemm_i8_topk_kernel<17>
             : kp <= 24 ? gemm_i8_topk_kernel<24> : gemm_i8_topk_kernel<32>;
    if (!set_smem_attr(reinterpret_cast<const void*>(k), kISmemTopk)) {
      set_error("route: cannot set dynamic shared memory size of the fused i8 GEMM");
      return OMNIMOE_ERR_CUDA;
    }
    k<<<g, 128 + 32 * kIEpiWarps, kISmemTopk, st>>>(mA, mB, a, ta);
    OMNI_CHECK_LAUNCH("gemm_i8_topk_kernel");
    if (fr) {
      fr->cand = ta.cand;
      fr->part = ta.part;
      fr->kp = kp;
      fr->counts = w.counts;
      fr->bad_x = w.bad_x;
    }
    // flagged rows: the fp64 kernel rewrites those tokens' logits (all columns), flagged
    // sub-key rows those columns (the epilogue then wrote every logit too); the selection
    // reads the logits wherever a flag applies
    OMNI_TRY(launch_exact_dd(d.dtype, x, sub, (int)d.d, NC, (int)L, logits, 1, w.bad_x, w.counts, st));
    return launch_exact_dd(d.dtype, x, sub, (int)d.d, NC, (int)L, logits, 2, w.bad_w, w.counts + 1, st);
  }
  if (fr) fr->kp = 0;
  if (CN == 1 && tuning().i8_persist) {
    const int64_t tiles = (int64_t)grid.x * grid.y;
    gemm_i8_persist_kernel<<<(int)std::min<int64_t>(tiles, num_sms()), 128 + 32 * kIEpiWarps, kISmemBytes, st>>>(mA, mB,
                                                                                                         a);
  } else if (CN == 1) {
    gemm_i8_exact_kernel<1><<<grid, 256, kISmemBytes, st>>>(mA, mB, a);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = kISmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CN;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = CN == 4 ? cudaLaunchKernelEx(&cfg, gemm_i8_exact_kernel<4>, mA, mB, a)
                            : cudaLaunchKernelEx(&cfg, gemm_i8_exact_kernel<2>, mA, mB, a);
    if (e != cudaSuccess) {
      set_error(std::string("gemm_i8_exact_kernel (cluster launch): ") + cudaGetErrorString(e));
      return OMNIMOE_ERR_CUDA;
    }
  }
  OMNI_CHECK_LAUNCH("gemm_i8_exact_kernel");
  // rows whose exponents do not fit 22 bits: exact fp64 path (no-ops when the lists are empty)
  OMNI_TRY(launch_exact_dd(d.dtype, x, sub, (int)d.d, NC, (int)L, logits, 1, w.bad_x, w.counts, st));
  return launch_exact_dd(d.dtype, x, sub, (int)d.d, NC, (int)L, logits, 2, w.bad_w, w.counts + 1, st);
}

}  // namespace omni
