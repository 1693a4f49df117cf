// Device twin of synth/__init__.py: the seeded counter-based input generator.
// Holds no arithmetic of the OmniMoE method; it only fills buffers with
// (seed, tensor id, index) -> v * 2^-e draws, bit-identical to the numpy
// implementation (tests/test_gpu_parity.py::test_synth_device_matches_host checks this).  Built into
// synth/libsynth.so, separate from the product library.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int64_t draw(uint64_t seed, uint64_t tid, uint64_t index, int mode) {
  uint64_t key = ((seed & 0xFF) << 56) ^ ((tid & 0xFF) << 48) ^ index;
  uint64_t h = splitmix64(key);
  if (mode == 1) return (int64_t)(h % 9ull) - 4;
  uint64_t s = (h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + (h >> 48);
  return (int64_t)s - 131070;
}

__global__ void fill_kernel(uint64_t seed, uint64_t tid, uint64_t base, uint64_t n, int e, int mode,
                            int out_bf16, void* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float f = ldexpf((float)draw(seed, tid, base + i, mode), -e);
    if (out_bf16) {
      uint32_t b = __float_as_uint(f);
      b = (b + 0x7FFFu + ((b >> 16) & 1u)) >> 16;
      reinterpret_cast<uint16_t*>(out)[i] = (uint16_t)b;
    } else {
      reinterpret_cast<float*>(out)[i] = f;
    }
  }
}

}  // namespace

// Element i of `out` gets draw index base + i: a row shard of a tensor is the
// same numbers as the corresponding rows of the whole tensor.
extern "C" int synth_fill(uint64_t seed, uint64_t tensor_id, uint64_t base, uint64_t n, int e, int mode,
                          int out_bf16, void* out, cudaStream_t stream) {
  if (n == 0) return 0;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  fill_kernel<<<blocks, 256, 0, stream>>>(seed, tensor_id, base, n, e, mode, out_bf16, out);
  return (int)cudaGetLastError();
}
