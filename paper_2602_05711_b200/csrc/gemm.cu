// tcgen05 GEMM engine for sm_100a (router sub-key scoring a1, shared MLP a7/a8).
//
// Persistent: one CTA per SM walks 128 x 256 output tiles (static round-robin); the fp32
// tile accumulates in one of two 256-column TMEM buffers so that the epilogue of tile i
// overlaps the MMAs of tile i+1 (tfull / tempty mbarriers between the roles):
//   warp 0 (one lane)  TMA producer: 2-D cp.async.bulk.tensor loads of A (128x64)
//                      and B (2 x 128x64) bf16 boxes, 128B swizzle, into a
//                      kStages-deep SMEM ring guarded by full/empty mbarriers;
//   warp 1 (one lane)  MMA issuer: 4 x tcgen05.mma.cta_group::1.kind::f16
//                      (M=128, N=256, K=16) per 64-wide K block, accumulator in
//                      TMEM (256 columns); tcgen05.commit frees the SMEM slot;
//   warp 2             TMEM allocator;
//   warps 4..11        epilogue (two per TMEM lane quarter, one column half each):
//                      tcgen05.ld 32x32b.x32 -> registers -> fused
//                      epilogue (fp32 store | SiLU(gate)*up -> bf16 | +addend -> bf16).
#include <mutex>

#include "gemm.cuh"
#include "tcgen05.cuh"

namespace omni {
namespace {
using namespace tc;

constexpr int BM = 128, BN = 256, BK = 64, kStages = 4;
constexpr int kABytes = BM * BK * 2;        // 16 KB
constexpr int kBBytes = BN * BK * 2;        // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kEpiWarps = 8;    // epilogue warps 4..11 (two per TMEM lane quarter)
constexpr int kGateStage = 16;  // EPI_GATED: gates staged per row and half tile (K/N x 128 on average)
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kSmemGated = kSmemBytes + kEpiWarps * 32 * kGateStage * 4;
static_assert(kSmemGated <= 232448, "EPI_GATED shared memory");

// instruction descriptor, kind::f16: D=f32, A=B=bf16, both K-major, M=128, N=256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

constexpr uint32_t kIdescBmn = kIdesc | (1u << 16);  // b_major = MN

template <int EPI, bool BMN = false>
__global__ void __launch_bounds__(128 + 32 * kEpiWarps, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmB2, GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [2]: MMA -> epilogue
  uint64_t* tempty = tfull + 2;        // [2]: epilogue -> MMA (4 warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // derived from smem_raw itself so that the compiler emits LDS/STS (not generic accesses)
  float* gated_smem = reinterpret_cast<float*>(smem_raw + (smem - smem_raw) + kStages * kStageBytes + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_kb = (args.K + BK - 1) / BK;
  const int ncols = (EPI == EPI_SWIGLU) ? BN / 2 : BN;
  const int n_nt = (args.N + ncols - 1) / ncols;
  const int n_mt = (args.M + BM - 1) / BM;
  const int n_tiles = n_nt * n_mt;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (one K-block ring across all tiles) ----------------
    int g = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x)
    for (int kb = 0; kb < num_kb; ++kb, ++g) {
      const int m0 = (args.m_fast ? t % n_mt : t / n_nt) * BM, nt = args.m_fast ? t / n_mt : t % n_nt;
      const int s = g % kStages;
      const uint32_t ph = (g / kStages) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], kStageBytes);
      tma_load_2d(&tmA, &full[s], sA + s * kABytes, kb * BK, m0);
      if (EPI == EPI_SWIGLU) {
        tma_load_2d(&tmB, &full[s], sB + s * kBBytes, kb * BK, nt * (BN / 2));
        tma_load_2d(&tmB2, &full[s], sB + s * kBBytes + kBBytes / 2, kb * BK, nt * (BN / 2));
      } else if (BMN) {  // four [64 K][64 N] boxes of the row-major [K][N] operand
#pragma unroll
        for (int i = 0; i < BN / 64; ++i)
          tma_load_2d(&tmB, &full[s], sB + s * kBBytes + i * (kBBytes / (BN / 64)), nt * BN + 64 * i, kb * BK);
      } else {
        const int kB = args.b_kwrap ? (kb * BK) % args.b_kwrap : kb * BK;
        tma_load_2d(&tmB, &full[s], sB + s * kBBytes, kB, nt * BN);
        tma_load_2d(&tmB, &full[s], sB + s * kBBytes + kBBytes / 2, kB, nt * BN + BN / 2);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread) ----------------
    int g = 0, it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      mbar_wait(&tempty[b], ((it >> 1) & 1) ^ 1);  // the epilogue has drained this buffer
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc = tmem + (uint32_t)(b * BN);
      for (int kb = 0; kb < num_kb; ++kb, ++g) {
        const int s = g % kStages;
        const uint32_t ph = (g / kStages) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(sA + s * kABytes), b0 = smem_u32(sB + s * kBBytes);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          if (BMN)  // K = 16 spans two 8-row swizzle atoms (2 KB); MN blocks 8 KB apart
            umma_f16(acc, sw128_desc(a0 + k * 32), sw128_desc_mn(b0 + k * 2048, kBBytes / (BN / 64)), kIdescBmn,
                     (kb | k) != 0);
          else
            umma_f16(acc, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), kIdesc, (kb | k) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(&tfull[b]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (TMEM -> registers -> global) ----------------
    // kEpiWarps = 8: warp 4 + e reads TMEM lane quarter e % 4 (its hardware-fixed lanes)
    // and column half e / 4 of the tile, two warps per SM sub-partition so that one
    // warp's TMEM/global latency overlaps the other's arithmetic
    const int e = warp - 4, q = e & 3, h = e >> 2;
    const int nchunk = ((EPI == EPI_SWIGLU) ? BN / 2 : BN) / 32;
    const int c_lo = h * nchunk / 2, c_hi = (h + 1) * nchunk / 2;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
    const int m0 = (args.m_fast ? t % n_mt : t / n_nt) * BM, nt = args.m_fast ? t / n_mt : t % n_nt;
    const int b = it & 1;
    if (EPI != EPI_GATED) {
      mbar_wait(&tfull[b], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const int row = m0 + q * 32 + lane;
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN);
    const bool row_ok = row < args.M;
    if (EPI == EPI_SWIGLU) {
      __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(args.out);
#pragma unroll 1
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t g[32], u[32];
        tmem_ld32(tbase + c * 32, g);
        tmem_ld32(tbase + BN / 2 + c * 32, u);
        const int col0 = nt * (BN / 2) + c * 32;
        if (!row_ok) continue;
        __nv_bfloat16* dst = H + (size_t)row * (args.h_split ? 2 * args.N : args.N) + col0;
        if (col0 + 32 <= args.N && (args.N % 8) == 0) {
          uint32_t p[16], pl[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float h0 = silu_f(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]);
            const float h1 = silu_f(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]);
            p[i] = pack_bf16x2(h0, h1);
            pl[i] = pack_bf16x2(h0 - __uint_as_float(p[i] << 16), h1 - __uint_as_float(p[i] & 0xFFFF0000u));
          }
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int i = 0; i < 4; ++i) d4[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
          if (args.h_split) {
            uint4* l4 = reinterpret_cast<uint4*>(dst + args.N);
#pragma unroll
            for (int i = 0; i < 4; ++i) l4[i] = make_uint4(pl[4 * i], pl[4 * i + 1], pl[4 * i + 2], pl[4 * i + 3]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col0 + i < args.N) {
              const float h = silu_f(__uint_as_float(g[i])) * __uint_as_float(u[i]);
              const __nv_bfloat16 hi = __float2bfloat16_rn(h);
              dst[i] = hi;
              if (args.h_split) dst[args.N + i] = __float2bfloat16_rn(h - __bfloat162float(hi));
            }
        }
      }
    } else if (EPI == EPI_GATED) {
      // this row's 128-column half tile: 4 mask words, one prefix count, and its gates
      // (about K/N x 128 of them) staged in shared memory -- two dependent global round
      // trips per tile, issued before the accumulator wait so they overlap the tile's MMAs
      __nv_bfloat16* A = reinterpret_cast<__nv_bfloat16*>(args.out);
      float* gsm = gated_smem + e * 32 * kGateStage;
      uint4 bits = make_uint4(0u, 0u, 0u, 0u);
      const float* gc = nullptr;
      const int w0 = nt * (BN / 32);
      if (row_ok && w0 < args.mask_words) {
        const uint4* m4 = reinterpret_cast<const uint4*>(args.mask + (size_t)row * args.mask_words + w0);
        const uint4 lo = m4[0], hi = m4[1];
        const uint4 mine = h ? hi : lo;
        bits = mine;
        const int before = h ? __popc(lo.x) + __popc(lo.y) + __popc(lo.z) + __popc(lo.w) : 0;
        const int cnt = __popc(bits.x) + __popc(bits.y) + __popc(bits.z) + __popc(bits.w);
        gc = args.gate_c + (size_t)row * args.gate_ld + args.mask_prefix[(size_t)row * (args.mask_words / 8) + nt] +
             before;
        // unconditional (clamped) loads so that all kGateStage of them are in flight at once
        float gv[kGateStage];
#pragma unroll
        for (int j = 0; j < kGateStage; ++j) gv[j] = gc[cnt > 0 ? min(j, cnt - 1) : 0];
#pragma unroll
        for (int j = 0; j < kGateStage; ++j) gsm[j * 32 + lane] = gv[j];
      }
      mbar_wait(&tfull[b], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      int k = 0;
#pragma unroll 1
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        const int col0 = nt * BN + c * 32;
        if (!row_ok || col0 >= args.out_ld) continue;
        const int j = c - c_lo;
        const uint32_t bw = j == 0 ? bits.x : j == 1 ? bits.y : j == 2 ? bits.z : bits.w;
        uint32_t p[16];
        if (bw == 0) {
#pragma unroll
          for (int i = 0; i < 16; ++i) p[i] = 0u;
        } else {
          // branch-free: every lane evaluates all 32 columns (the selected columns differ
          // per lane, so a per-column branch would serialise the warp); the rank of column
          // i among the chunk's set bits indexes the staged gates
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const bool sel = (bw >> i) & 1u;
            const int kk = k + __popc(bw & ((1u << i) - 1u));
            float g = gsm[min(kk, kGateStage - 1) * 32 + lane];
            if (sel && kk >= kGateStage) g = gc[kk];
            const float z = __uint_as_float(r[i]);
            const float a = args.act == OMNIMOE_IDENTITY ? z : __fdividef(z, 1.0f + __expf(-z));
            v[i] = sel ? g * a : 0.f;
          }
          k += __popc(bw);
#pragma unroll
          for (int i = 0; i < 16; ++i) p[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
        }
        __nv_bfloat16* dst = A + (size_t)row * args.out_ld + col0;
#pragma unroll
        for (int i = 0; i < 4; ++i)  // out_ld % 8 == 0: whole uint4s, also in a ragged tail
          if (col0 + 8 * i < args.out_ld)
            reinterpret_cast<uint4*>(dst)[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
      }
    } else {
#pragma unroll 1
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + c * 32, r);
        const int col0 = nt * BN + c * 32;
        if (!row_ok || col0 >= args.N) continue;
        const bool vec = (col0 + 32 <= args.N) && (args.N % 8) == 0;
        if (EPI == EPI_F32) {
          float* dst = args.out_f32 + (size_t)row * args.N + col0;
          if (vec) {
            float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              d4[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                  __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < args.N) dst[i] = __uint_as_float(r[i]);
          }
        } else {  // EPI_ADD -> bf16
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)row * args.N + col0;
          const float* add = args.addend ? args.addend + (size_t)row * args.N + col0 : nullptr;
          if (vec) {
            float a[32];
            if (add) {
              const float4* a4 = reinterpret_cast<const float4*>(add);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float4 t = a4[i];
                a[4 * i] = t.x; a[4 * i + 1] = t.y; a[4 * i + 2] = t.z; a[4 * i + 3] = t.w;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) a[i] = 0.f;
            }
            uint32_t p[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              p[i] = pack_bf16x2(__uint_as_float(r[2 * i]) + a[2 * i],
                                 __uint_as_float(r[2 * i + 1]) + a[2 * i + 1]);
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int i = 0; i < 4; ++i) d4[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < args.N) dst[i] = __float2bfloat16_rn(__uint_as_float(r[i]) + (add ? add[i] : 0.f));
          }
        }
      }
    }
    // this warp's TMEM lanes of buffer b are read: release it to the MMA issuer
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[b])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
}

bool make_map(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t k, uint32_t box_rows) {
  return tc::make_map_2d(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, rows, k, BK, box_rows);
}

template <int EPI, bool BMN = false>
omnimoe_status launch_tc(const void* A, const void* B, const GemmArgs& a, cudaStream_t st) {
  if (!set_smem_attr(reinterpret_cast<const void*>(gemm_tc_kernel<EPI, BMN>),
                     EPI == EPI_GATED ? kSmemGated : kSmemBytes)) {
    set_error("gemm: cannot set dynamic shared memory size");
    return OMNIMOE_ERR_CUDA;
  }
  CUtensorMap mA, mB, mB2;
  bool ok = make_map(&mA, A, a.M, a.K, BM);
  if (EPI == EPI_SWIGLU) {
    ok = ok && make_map(&mB, B, a.N, a.K, BN / 2);
    ok = ok && make_map(&mB2, static_cast<const char*>(B) + (size_t)a.N * a.K * 2, a.N, a.K, BN / 2);
  } else if (BMN) {
    ok = ok && make_map(&mB, B, (uint64_t)(a.b_rows > 0 ? a.b_rows : a.K), a.N, 64);
    mB2 = mB;
  } else {
    if (a.b_kwrap && (a.b_kwrap % BK != 0 || a.K % a.b_kwrap != 0)) {
      set_error("gemm: b_kwrap must be a multiple of 64 dividing K");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
    ok = ok && make_map(&mB, B, a.N, a.b_kwrap ? a.b_kwrap : a.K, BN / 2);
    mB2 = mB;
  }
  if (!ok) {
    set_error("gemm: cuTensorMapEncodeTiled failed (alignment: K % 8 == 0, 16-byte base)");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  const int ncols = (EPI == EPI_SWIGLU) ? BN / 2 : BN;
  const int64_t tiles = (int64_t)((a.N + ncols - 1) / ncols) * ((a.M + BM - 1) / BM);
  GemmArgs ka = a;
  if (ka.m_fast < 0) {
    // m fastest: the CTAs in flight share a few B tiles and sweep all of A, so B is read
    // from HBM once when A stays in L2 (C4's Z = x W^T: A = 8 MB, B = 210 MB).
    const double a_bytes = (double)a.M * a.K * 2, b_bytes = (double)a.N * a.K * 2 * (EPI == EPI_SWIGLU ? 2 : 1);
    ka.m_fast = (a_bytes < b_bytes && a_bytes <= 48.0 * (1 << 20)) ? 1 : 0;
  }
  if (tuning().gemm_mfast >= 0) ka.m_fast = tuning().gemm_mfast;
  gemm_tc_kernel<EPI, BMN><<<(int)std::min<int64_t>(tiles, num_sms()), 128 + 32 * kEpiWarps,
                        EPI == EPI_GATED ? kSmemGated : kSmemBytes, st>>>(
      mA, mB, mB2, ka);
  OMNI_CHECK_LAUNCH("gemm_tc_kernel");
  return OMNIMOE_OK;
}

// ---------------------------------------------------------------------------
// fp32 SIMT GEMM (OMNIMOE_F32 correctness mode): 64x64 tile, 256 threads, 4x4 per thread.
template <int EPI>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A,
                                                       const float* __restrict__ B, GemmArgs a) {
  __shared__ float sa[16][64 + 4], sb[2][16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int nb = (EPI == EPI_SWIGLU) ? 2 : 1;
  float acc[2][4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      int r = i / 16, kk = i % 16;
      int m = m0 + r, k = k0 + kk;
      sa[kk][r] = (m < a.M && k < a.K) ? A[(size_t)m * a.K + k] : 0.f;
      for (int b = 0; b < nb; ++b) {
        int n = n0 + r;
        sb[b][kk][r] = (n < a.N && k < a.K) ? B[((size_t)b * a.N + n) * a.K + k] : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk)
      for (int b = 0; b < nb; ++b)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[b][i][j] = fmaf(sa[kk][ty * 4 + i], sb[b][kk][tx * 4 + j], acc[b][i][j]);
    __syncthreads();
  }
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m >= a.M || n >= a.N) continue;
      size_t o = (size_t)m * a.N + n;
      if (EPI == EPI_F32) a.out_f32[o] = acc[0][i][j];
      else if (EPI == EPI_SWIGLU) reinterpret_cast<float*>(a.out)[o] = silu_f(acc[0][i][j]) * acc[1][i][j];
      else reinterpret_cast<float*>(a.out)[o] = acc[0][i][j] + (a.addend ? a.addend[o] : 0.f);
    }
}

}  // namespace

namespace tc {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D row-major tensor [rows][cols], box [box_rows][box_cols] with 128-byte swizzle
// (box_cols * elem_bytes must be 128).
bool make_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int elem_bytes, const void* ptr,
                 uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace tc

omnimoe_status gemm_bf16(int epi, const void* A, const void* B, const GemmArgs& a, cudaStream_t st) {
  if (a.M == 0 || a.N == 0) return OMNIMOE_OK;
  switch (epi) {
    case EPI_F32: return a.b_mn ? launch_tc<EPI_F32, true>(A, B, a, st) : launch_tc<EPI_F32>(A, B, a, st);
    case EPI_SWIGLU: return launch_tc<EPI_SWIGLU>(A, B, a, st);
    case EPI_ADD: return launch_tc<EPI_ADD>(A, B, a, st);
    case EPI_GATED: return launch_tc<EPI_GATED>(A, B, a, st);
  }
  return OMNIMOE_ERR_UNSUPPORTED;
}

omnimoe_status gemm_f32(int epi, const float* A, const float* B, const GemmArgs& a, cudaStream_t st) {
  if (a.M == 0 || a.N == 0) return OMNIMOE_OK;
  dim3 grid((a.N + 63) / 64, (a.M + 63) / 64);
  switch (epi) {
    case EPI_F32: gemm_f32_kernel<EPI_F32><<<grid, 256, 0, st>>>(A, B, a); break;
    case EPI_SWIGLU: gemm_f32_kernel<EPI_SWIGLU><<<grid, 256, 0, st>>>(A, B, a); break;
    case EPI_ADD: gemm_f32_kernel<EPI_ADD><<<grid, 256, 0, st>>>(A, B, a); break;
    default: return OMNIMOE_ERR_UNSUPPORTED;
  }
  OMNI_CHECK_LAUNCH("gemm_f32_kernel");
  return OMNIMOE_OK;
}

}  // namespace omni
