// TMA gather4 ceiling for pass V's access pattern: random 128-byte pieces from a 64 MB
// L2-resident table moved into shared memory by `cp.async.bulk.tensor.2d...tile::gather4`
// (4 rows per instruction, no registers held while in flight), then consumed from shared
// memory with the pass-V lane layout (8 pieces x 4 quarters per round, bf16 -> fp32 FMA).
// One producer warp (lanes 0..7 each issue one gather4 of a 32-piece stage) and C consumer
// warps per CTA, an S-stage ring with full / empty mbarriers.  Compared with the LDG.256
// ceiling of tools/l2_ceiling.cu (18.8 TB/s for 128-byte pieces).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_gather tools/tma_gather.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void gather4(const CUtensorMap* m, uint64_t* bar, void* dst, int col, int4 r) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(col), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su32(bar))
      : "memory");
}

constexpr int kStageBytes = 32 * 128;  // 32 pieces

// NP independent pipes per CTA, each = one producer warp + CP consumer warps + its own ring of
// SP stages (a producer never runs more than SP stages ahead of its own consumers, so the
// mbarrier parities stay exact); CTA b, pipe p handles stages k = p, p + NP, ... of the CTA's n
template <int SP, int CP, int NP>
__global__ void __launch_bounds__(32 * NP * (CP + 1), 1)
    tma_gather(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx, int n, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pipe = warp / (CP + 1), role = warp % (CP + 1);  // role CP: producer
  uint8_t* ring = smem + pipe * SP * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NP * SP * kStageBytes) + pipe * 2 * SP;
  uint64_t* empty = full + SP;
  if (role == 0 && lane == 0) {
    for (int s = 0; s < SP; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CP); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int* my = idx + (size_t)blockIdx.x * n * 32;
  const int nk = (n - pipe + NP - 1) / NP;  // this pipe's stages: j = 0..nk-1 -> k = pipe + NP j
  if (role == CP) {
    constexpr int D = 8;
    int4 rg[D];
#pragma unroll
    for (int j = 0; j < D; ++j)
      rg[j] = (j < nk && lane < 8) ? reinterpret_cast<const int4*>(my + (size_t)(pipe + NP * j) * 32)[lane] : make_int4(0, 0, 0, 0);
    for (int j0 = 0; j0 < nk; j0 += D) {
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const int j = j0 + u;
        if (j < nk) {
          const int4 cur = rg[u];
          if (j + D < nk && lane < 8) rg[u] = reinterpret_cast<const int4*>(my + (size_t)(pipe + NP * (j + D)) * 32)[lane];
          const int s = j % SP;
          if (j >= SP) mbar_wait(&empty[s], ((j / SP) - 1) & 1);
          if (lane == 0) mbar_expect_tx(&full[s], kStageBytes);
          __syncwarp();
          if (lane < 8) gather4(&tm, &full[s], ring + s * kStageBytes + lane * 512, 0, cur);
        }
      }
    }
  } else {  // consumers: each reads a CP-th of every stage, lane = (g8 piece sub-slot, c4 quarter)
    const int c4 = lane & 3, g8 = lane >> 2;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    for (int j = 0; j < nk; ++j) {
      const int s = j % SP;
      mbar_wait(&full[s], (j / SP) & 1);
      const uint8_t* st = ring + s * kStageBytes;
#pragma unroll
      for (int r = role; r < 4; r += CP) {
        const uint4* p = reinterpret_cast<const uint4*>(st + (r * 8 + g8) * 128 + c4 * 32);
        uint4 u0 = p[0], u1 = p[1];
        uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
        const float a = 1.0f + r;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[2 * i] = fmaf(a, __uint_as_float(w[i] << 16), acc[2 * i]);
          acc[2 * i + 1] = fmaf(a, __uint_as_float(w[i] & 0xffff0000u), acc[2 * i + 1]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) t += acc[i];
    if (t == 1234.5f) sink[0] = t;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int SP, int CP, int NP>
double run(const CUtensorMap& tm, const int* idx, int n, int sms, float* sink, int per_sm) {
  const size_t smem = NP * SP * (kStageBytes + 16);
  auto k = tma_gather<SP, CP, NP>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  const int blocks = sms * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<blocks, 32 * NP * (CP + 1), smem>>>(tm, idx, n, sink);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(cudaGetLastError())); return -1; }
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) k<<<blocks, 32 * NP * (CP + 1), smem>>>(tm, idx, n, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 5.0 * blocks * (double)n * kStageBytes;
  return bytes / (ms * 1e-3) / 1e9;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rows = 1 << 19;  // 512K x 128 B = 64 MB
  uint8_t* tab;
  CK(cudaMalloc(&tab, (size_t)rows * 128));
  CK(cudaMemset(tab, 1, (size_t)rows * 128));
  const int n = 2048;  // stages per CTA (64K pieces, 8 MB)
  const int max_blocks = sms * 4;
  std::vector<int> h((size_t)max_blocks * n * 32);
  uint64_t st = 88172645463325252ull;
  for (auto& v : h) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; v = (int)(st % rows); }
  int* idx;
  CK(cudaMalloc(&idx, h.size() * 4));
  CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  float* sink;
  CK(cudaMalloc(&sink, 4));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<EncodeFn>(fp);
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows}, strides[1] = {128};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  // correctness: one CTA, one stage, compare smem contents is implicit (sink); rate sweep:
  printf("{\"sms\": %d", sms);
#define RUN(SP, CP, NP, P) printf(", \"S%d_C%d_N%d_P%d\": %.0f", SP, CP, NP, P, run<SP, CP, NP>(tm, idx, n, sms, sink, P)); fflush(stdout);
  RUN(6, 1, 8, 1) RUN(4, 1, 12, 1) RUN(3, 1, 16, 1) RUN(2, 1, 16, 2) RUN(4, 1, 10, 1) RUN(6, 1, 4, 2) RUN(3, 1, 8, 2)
  RUN(2, 1, 12, 2) RUN(3, 1, 4, 4) RUN(2, 1, 6, 4)
  printf("}\n");
  return 0;
}
