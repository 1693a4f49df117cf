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
//   warps 4..7         epilogue: tcgen05.ld 32x32b.x32 -> registers -> fused
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
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

// instruction descriptor, kind::f16: D=f32, A=B=bf16, both K-major, M=128, N=256
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

template <int EPI>
__global__ void __launch_bounds__(256, 1)
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

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_kb = (args.K + BK - 1) / BK;
  const int ncols = (EPI == EPI_SWIGLU) ? BN / 2 : BN;
  const int n_nt = (args.N + ncols - 1) / ncols;
  const int n_tiles = n_nt * ((args.M + BM - 1) / BM);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
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
      const int m0 = (t / n_nt) * BM, nt = t % n_nt;
      const int s = g % kStages;
      const uint32_t ph = (g / kStages) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], kStageBytes);
      tma_load_2d(&tmA, &full[s], sA + s * kABytes, kb * BK, m0);
      if (EPI == EPI_SWIGLU) {
        tma_load_2d(&tmB, &full[s], sB + s * kBBytes, kb * BK, nt * (BN / 2));
        tma_load_2d(&tmB2, &full[s], sB + s * kBBytes + kBBytes / 2, kb * BK, nt * (BN / 2));
      } else {
        tma_load_2d(&tmB, &full[s], sB + s * kBBytes, kb * BK, nt * BN);
        tma_load_2d(&tmB, &full[s], sB + s * kBBytes + kBBytes / 2, kb * BK, nt * BN + BN / 2);
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
        for (int k = 0; k < BK / 16; ++k)
          umma_f16(acc, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), kIdesc, (kb | k) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(&tfull[b]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (TMEM -> registers -> global) ----------------
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
    const int m0 = (t / n_nt) * BM, nt = t % n_nt;
    const int b = it & 1;
    mbar_wait(&tfull[b], (it >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp - 4;  // TMEM lane quarter == warp id % 4
    const int row = m0 + q * 32 + lane;
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN);
    const bool row_ok = row < args.M;
    if (EPI == EPI_SWIGLU) {
      __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(args.out);
#pragma unroll 1
      for (int c = 0; c < BN / 2 / 32; ++c) {
        uint32_t g[32], u[32];
        tmem_ld32(tbase + c * 32, g);
        tmem_ld32(tbase + BN / 2 + c * 32, u);
        const int col0 = nt * (BN / 2) + c * 32;
        if (!row_ok) continue;
        __nv_bfloat16* dst = H + (size_t)row * args.N + col0;
        if (col0 + 32 <= args.N && (args.N % 8) == 0) {
          uint32_t p[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float g0 = __uint_as_float(g[2 * i]), g1 = __uint_as_float(g[2 * i + 1]);
            p[i] = pack_bf16x2(silu_f(g0) * __uint_as_float(u[2 * i]),
                               silu_f(g1) * __uint_as_float(u[2 * i + 1]));
          }
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int i = 0; i < 4; ++i) d4[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
        } else {
          for (int i = 0; i < 32 && col0 + i < args.N; ++i)
            dst[i] = __float2bfloat16_rn(silu_f(__uint_as_float(g[i])) * __uint_as_float(u[i]));
        }
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
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
            for (int i = 0; i < 32 && col0 + i < args.N; ++i) dst[i] = __uint_as_float(r[i]);
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
            for (int i = 0; i < 32 && col0 + i < args.N; ++i)
              dst[i] = __float2bfloat16_rn(__uint_as_float(r[i]) + (add ? add[i] : 0.f));
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

template <int EPI>
omnimoe_status launch_tc(const void* A, const void* B, const GemmArgs& a, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_tc_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemBytes) != cudaSuccess) {
      set_error("gemm: cannot set dynamic shared memory size");
      return OMNIMOE_ERR_CUDA;
    }
    attr_set = true;
  }
  CUtensorMap mA, mB, mB2;
  bool ok = make_map(&mA, A, a.M, a.K, BM);
  if (EPI == EPI_SWIGLU) {
    ok = ok && make_map(&mB, B, a.N, a.K, BN / 2);
    ok = ok && make_map(&mB2, static_cast<const char*>(B) + (size_t)a.N * a.K * 2, a.N, a.K, BN / 2);
  } else {
    ok = ok && make_map(&mB, B, a.N, a.K, BN / 2);
    mB2 = mB;
  }
  if (!ok) {
    set_error("gemm: cuTensorMapEncodeTiled failed (alignment: K % 8 == 0, 16-byte base)");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  const int ncols = (EPI == EPI_SWIGLU) ? BN / 2 : BN;
  const int64_t tiles = (int64_t)((a.N + ncols - 1) / ncols) * ((a.M + BM - 1) / BM);
  gemm_tc_kernel<EPI><<<(int)std::min<int64_t>(tiles, kSMs), 256, kSmemBytes, st>>>(mA, mB, mB2, a);
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
    case EPI_F32: return launch_tc<EPI_F32>(A, B, a, st);
    case EPI_SWIGLU: return launch_tc<EPI_SWIGLU>(A, B, a, st);
    case EPI_ADD: return launch_tc<EPI_ADD>(A, B, a, st);
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
