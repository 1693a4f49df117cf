// Phase-0 microbenchmarks that bound the a6 (expert) kernel on this B200:
//   hbm_read     : streaming 128-bit loads over a buffer >> L2
//   l2_gather    : warp-per-row random 4 KB row reads from an L2-resident table
//   red_scatter  : warp-per-row red.global.add.v4.f32 of 8 KB fp32 rows into
//                  random rows of a table (L2-resident and > L2)
//   ffma         : fp32 FMA issue rate (scalar fmaf)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void hbm_read(const uint4* __restrict__ p, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

// rows of row_bytes; each warp reads n_per_warp random rows
__global__ void l2_gather(const uint4* __restrict__ tab, int nrows, int row_vec, int n_per_warp, uint4* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int k = 0; k < n_per_warp; ++k) {
    uint32_t r = hash32(gw * 7919u + k) % nrows;
    const uint4* row = tab + (size_t)r * row_vec;
    for (int j = lane; j < row_vec; j += 32) {
      uint4 v = row[j];
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

__global__ void red_scatter(float* __restrict__ tab, int nrows, int row_f, int n_per_warp) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int k = 0; k < n_per_warp; ++k) {
    uint32_t r = hash32(gw * 7919u + k) % nrows;
    float* row = tab + (size_t)r * row_f;
    const float a = 1e-3f * (k + 1);
    for (int j = lane * 4; j < row_f; j += 128)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + j), "f"(a), "f"(a), "f"(a), "f"(a) : "memory");
  }
}

__global__ void ffma_rate(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, c5 = 0.f, c6 = 0.f, c7 = 0.f;
  for (int i = 0; i < iters; ++i) {
    c0 = fmaf(a, b, c0); c1 = fmaf(a, b, c1); c2 = fmaf(a, b, c2); c3 = fmaf(a, b, c3);
    c4 = fmaf(a, b, c4); c5 = fmaf(a, b, c5); c6 = fmaf(a, b, c6); c7 = fmaf(a, b, c7);
  }
  float s = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
  if (s == 1234.5f) out[0] = s;
}


// 128-byte pieces (8 lanes x 16 B) at byte offset `off` of random rows: the access
// pattern of a slice-major pass over an expert table (4 pieces per warp instruction)
__global__ void piece_gather(const uint4* __restrict__ tab, int nrows, int row_vec, int off_vec, int n_per_warp,
                             uint32_t salt, uint4* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll 4
  for (int k = 0; k < n_per_warp; k += 4) {
    uint32_t r = hash32((gw * 7919u + k + (lane >> 3)) ^ salt) % nrows;
    uint4 v = tab[(size_t)r * row_vec + off_vec + (lane & 7)];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

// 64-byte pieces (4 lanes x 16 B), 8 per warp instruction
__global__ void piece64_gather(const uint4* __restrict__ tab, int nrows, int n_per_warp, uint32_t salt, uint4* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll 4
  for (int k = 0; k < n_per_warp; k += 8) {
    uint32_t r = hash32((gw * 7919u + k + (lane >> 2)) ^ salt) & (nrows - 1);
    uint4 v = tab[(size_t)r * 4 + (lane & 3)];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

// 32-byte pieces (2 lanes x 16 B), 16 per warp instruction
__global__ void piece32_gather(const uint4* __restrict__ tab, int nrows, int n_per_warp, uint32_t salt, uint4* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll 4
  for (int k = 0; k < n_per_warp; k += 16) {
    uint32_t r = hash32((gw * 7919u + k + (lane >> 1)) ^ salt) & (nrows - 1);
    uint4 v = tab[(size_t)r * 2 + (lane & 1)];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

template <class F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("{\"sms\": %d, \"l2_bytes\": %d", sms, l2);
  uint4* sink; CK(cudaMalloc(&sink, 64));
  // HBM streaming read, 4 GiB
  size_t hb = size_t(4) << 30;
  uint4* big; CK(cudaMalloc(&big, hb)); CK(cudaMemset(big, 1, hb));
  float ms = time_ms([&] { hbm_read<<<sms * 8, 512>>>(big, hb / 16, sink); });
  printf(", \"hbm_read_gbs\": %.1f", hb / ms / 1e6);
  // L2 gather: 64 MB table of 4 KB rows
  const int row_b = 4096, nrows = (64 << 20) / row_b;
  int nw = sms * 64;
  for (int npw : {64}) {
    ms = time_ms([&] { l2_gather<<<nw / 8, 256>>>(big, nrows, row_b / 16, npw, sink); });
    printf(", \"l2_gather_4KB_rows_gbs\": %.1f", (double)nw * npw * row_b / ms / 1e6);
  }
  // HBM gather: rows from the whole 4 GiB
  ms = time_ms([&] { l2_gather<<<nw / 8, 256>>>(big, (int)(hb / row_b), row_b / 16, 64, sink); });
  printf(", \"hbm_gather_4KB_rows_gbs\": %.1f", (double)nw * 64 * row_b / ms / 1e6);
  // red scatter of 8 KB fp32 rows (2048 floats): table of 64 MB (L2) and 134 MB / 512 MB
  for (size_t tb : {size_t(64) << 20, size_t(134) << 20, size_t(512) << 20}) {
    float* tab = reinterpret_cast<float*>(big);
    int rows = (int)(tb / 8192);
    ms = time_ms([&] { red_scatter<<<nw / 8, 256>>>(tab, rows, 2048, 16); });
    printf(", \"red_v4_scatter_8KB_rows_%zuMB_gbs\": %.1f", tb >> 20, (double)nw * 16 * 8192 / ms / 1e6);
  }

  // slice-pass pattern: 128 B pieces of random rows among 524288 rows of 4 KB (67 MB of lines)
  {
    const int prow = 524288, pnpw = 1024, pw = sms * 64;
    ms = time_ms([&] { piece_gather<<<pw / 8, 256>>>(big, prow, 256, 0, pnpw, 0u, sink); });
    printf(", \"l2_piece128_gather_67MB_gbs\": %.1f", (double)pw * pnpw * 128 / ms / 1e6);
    // the same over 1M rows (134 MB of lines: exceeds L2)
    ms = time_ms([&] { piece_gather<<<pw / 8, 256>>>(big, 1 << 20, 256, 0, pnpw, 0u, sink); });
    printf(", \"piece128_gather_134MB_gbs\": %.1f", (double)pw * pnpw * 128 / ms / 1e6);
    // a sweep of 32 slices (cold first touch of each slice), 4.2M pieces per slice
    const int npw2 = 4 * 1048576 / pw;
    ms = time_ms([&] {
      for (int s = 0; s < 32; ++s) piece_gather<<<pw / 8, 256>>>(big, prow, 256, s * 8, npw2, 77u * s, sink);
    }, 3);
    printf(", \"piece128_slice_sweep_gbs\": %.1f, \"piece128_slice_sweep_ms\": %.3f",
           (double)pw * npw2 * 32 * 128 / ms / 1e6, ms);

    // the same pieces packed contiguously (slice-major layout: 67 MB span, within TLB reach)
    ms = time_ms([&] { piece_gather<<<pw / 8, 256>>>(big, prow, 8, 0, pnpw, 0u, sink); });
    printf(", \"l2_piece128_packed_67MB_gbs\": %.1f", (double)pw * pnpw * 128 / ms / 1e6);
    ms = time_ms([&] {
      for (int s = 0; s < 32; ++s) piece_gather<<<pw / 8, 256>>>(big + (size_t)s * prow * 8, prow, 8, 0, npw2, 77u * s, sink);
    }, 3);
    printf(", \"piece128_packed_sweep_gbs\": %.1f, \"piece128_packed_sweep_ms\": %.3f",
           (double)pw * npw2 * 32 * 128 / ms / 1e6, ms);
    ms = time_ms([&] { piece64_gather<<<pw / 8, 256>>>(big, 1 << 20, pnpw * 2, 0u, sink); });
    printf(", \"l2_piece64_packed_67MB_gbs\": %.1f", (double)pw * pnpw * 2 * 64 / ms / 1e6);
    ms = time_ms([&] {
      for (int s = 0; s < 32; ++s) piece64_gather<<<pw / 8, 256>>>(big + (size_t)s * (1 << 20) * 4, 1 << 20, npw2 * 2, 77u * s, sink);
    }, 3);
    printf(", \"piece64_packed_sweep_gbs\": %.1f", (double)pw * npw2 * 2 * 32 * 64 / ms / 1e6);
    ms = time_ms([&] { piece32_gather<<<pw / 8, 256>>>(big, 1 << 20, pnpw * 4, 0u, sink); });
    printf(", \"l2_piece32_packed_33MB_gbs\": %.1f", (double)pw * pnpw * 4 * 32 / ms / 1e6);
    ms = time_ms([&] {
      for (int s = 0; s < 64; ++s) piece32_gather<<<pw / 8, 256>>>(big + (size_t)s * (1 << 20) * 2, 1 << 20, npw2 * 4, 77u * s, sink);
    }, 3);
    printf(", \"piece32_packed_sweep_gbs\": %.1f", (double)pw * npw2 * 4 * 64 * 32 / ms / 1e6);
    ms = time_ms([&] {
      for (int s = 0; s < 64; ++s) piece64_gather<<<pw / 8, 256>>>(big + (size_t)s * (1 << 19) * 4, 1 << 19, npw2 * 2, 77u * s, sink);
    }, 3);
    printf(", \"piece64_packed_sweep_33MB_gbs\": %.1f", (double)pw * npw2 * 2 * 64 * 64 / ms / 1e6);
  }
  // FFMA rate
  float* o; CK(cudaMalloc(&o, 64));
  const int iters = 4096;
  ms = time_ms([&] { ffma_rate<<<sms * 8, 256>>>(o, iters); });
  printf(", \"ffma_tflops\": %.1f", 2.0 * 8 * iters * (double)sms * 8 * 256 / ms / 1e9);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf(", \"clock_khz_attr\": %d}\n", clk);
  return 0;
}
