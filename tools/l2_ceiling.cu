// L2 -> SM gather ceiling on this B200, for the access patterns of the a6 kernels:
// random pieces of PB bytes (128: a pass-V slice piece; 4096: a pass-Z x row) from a
// 64 MB L2-resident table, read with 256-bit loads (LDG.E.256) by every lane, piece
// indices precomputed in global memory like the kernels' plans.  Sweeps the 256-bit
// loads in flight per lane (U) and the CTAs per SM (MINB via launch bounds) and prints
// one JSON object with the best rate per piece size -- the denominator bench.py uses
// for roofline.l2 (profiles/r2/l2_ceiling/).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/l2_ceiling tools/l2_ceiling.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s\n", cudaGetErrorString(e)); return 1; } } while (0)

struct U8 { uint32_t w[8]; };
__device__ __forceinline__ U8 ld256(const void* p) {
  U8 r;
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                 "=r"(r.w[7]) : "l"(p));
  return r;
}

// each warp handles n_per_warp pieces; PB / 32 lanes per piece-instruction slot
template <int PB, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
    gather(const uint8_t* __restrict__ tab, const int* __restrict__ idx, int n_per_warp, uint32_t* sink) {
  constexpr int LPP = PB >= 1024 ? 32 : PB / 32;      // lanes per piece in one instruction
  constexpr int PPI = 32 / LPP;                       // pieces per instruction
  constexpr int IPP = PB >= 1024 ? PB / 1024 : 1;     // instructions per piece
  const int lane = threadIdx.x & 31;
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int* my = idx + gw * n_per_warp;
  uint32_t acc = 0;
  for (int k = 0; k < n_per_warp; k += PPI * U / IPP) {
    U8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int inst = u % IPP, pc = u / IPP;  // instruction u covers part `inst` of piece group pc
      const int piece = k + pc * PPI + lane / LPP;
      const int r = my[piece < n_per_warp ? piece : 0];
      v[u] = ld256(tab + (size_t)r * PB + inst * 1024 + (lane % LPP) * 32);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc ^= v[u].w[i];
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int PB, int U, int MINB>
double run(const uint8_t* tab, const int* idx, int nrows, int sms, uint32_t* sink) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather<PB, U, MINB>, 256, 0);
  const int blocks = sms * per_sm, warps = blocks * 8;
  const long total = 4l << 30;  // 4 GB of pieces per run, split over the warps
  int n_per_warp = (int)(total / PB / warps);
  n_per_warp = (n_per_warp / 64 + 1) * 64;
  (void)nrows;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  gather<PB, U, MINB><<<blocks, 256>>>(tab, idx, n_per_warp, sink);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    gather<PB, U, MINB><<<blocks, 256>>>(tab, idx, n_per_warp, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return (double)warps * n_per_warp * PB / best / 1e6;  // GB/s
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t tab_bytes = 64ul << 20;
  uint8_t* tab; CK(cudaMalloc(&tab, tab_bytes)); CK(cudaMemset(tab, 1, tab_bytes));
  const size_t nidx = 64ul << 20;  // enough for every configuration's warps x pieces
  std::vector<int> h(nidx);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  uint32_t* sink; CK(cudaMalloc(&sink, 64));
  printf("{\"sms\": %d", sms);
  for (int pb : {128, 4096}) {
    const int nrows = (int)(tab_bytes / pb);
    for (size_t i = 0; i < nidx; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (int)(s % nrows);
    }
    int* idx; CK(cudaMalloc(&idx, nidx * 4)); CK(cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    double best = 0; const char* arg = "";
    auto note = [&](double g, const char* name) { printf(", \"pb%d_%s\": %.0f", pb, name, g); if (g > best) { best = g; arg = name; } };
    if (pb == 128) {
      note(run<128, 4, 2>(tab, idx, nrows, sms, sink), "U4_B2");
      note(run<128, 4, 3>(tab, idx, nrows, sms, sink), "U4_B3");
      note(run<128, 4, 4>(tab, idx, nrows, sms, sink), "U4_B4");
      note(run<128, 8, 2>(tab, idx, nrows, sms, sink), "U8_B2");
      note(run<128, 8, 3>(tab, idx, nrows, sms, sink), "U8_B3");
      note(run<128, 2, 6>(tab, idx, nrows, sms, sink), "U2_B6");
      note(run<128, 2, 8>(tab, idx, nrows, sms, sink), "U2_B8");
      note(run<128, 16, 1>(tab, idx, nrows, sms, sink), "U16_B1");
    } else {
      note(run<4096, 4, 4>(tab, idx, nrows, sms, sink), "U4_B4");
      note(run<4096, 8, 2>(tab, idx, nrows, sms, sink), "U8_B2");
      note(run<4096, 8, 3>(tab, idx, nrows, sms, sink), "U8_B3");
      note(run<4096, 16, 1>(tab, idx, nrows, sms, sink), "U16_B1");
      note(run<4096, 16, 2>(tab, idx, nrows, sms, sink), "U16_B2");
      note(run<4096, 4, 6>(tab, idx, nrows, sms, sink), "U4_B6");
      note(run<4096, 4, 8>(tab, idx, nrows, sms, sink), "U4_B8");
    }
    printf(", \"pb%d_best_gbs\": %.0f, \"pb%d_best\": \"%s\"", pb, best, pb, arg);
    cudaFree(idx);
  }
  printf("}\n");
  return 0;
}
