// Shared device/host helpers of the OmniMoE B200 library (sm_100a only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/omnimoe.h"
#include "tuning.cuh"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libomnimoe targets sm_100a only"
#endif

namespace omni {

// SM count of the current device, queried once per device (148 on B200): grids are
// sized in multiples of it (persistent kernels: one wave of resident CTAs)
int num_sms();
// cudaFuncSetAttribute(func, MaxDynamicSharedMemorySize, bytes), applied once per
// (kernel, device, size) behind a lock: safe for several devices and host threads
bool set_smem_attr(const void* func, int bytes);

// ---- host-side error state (thread-local, see omnimoe_last_error) ----------
void set_error(const std::string& msg);
void count_launch(int n = 1);
void reset_launch_count();

#define OMNI_CHECK_LAUNCH(what)                                                   \
  do {                                                                            \
    cudaError_t e__ = cudaGetLastError();                                         \
    if (e__ != cudaSuccess) {                                                     \
      ::omni::set_error(std::string(what) + ": " + cudaGetErrorString(e__));      \
      return OMNIMOE_ERR_CUDA;                                                    \
    }                                                                             \
    ::omni::count_launch();                                                       \
  } while (0)

#define OMNI_TRY(expr)                        \
  do {                                        \
    omnimoe_status s__ = (expr);              \
    if (s__ != OMNIMOE_OK) return s__;        \
  } while (0)

// ---- workspace carving ------------------------------------------------------
struct Carver {
  char* base;
  size_t used = 0;
  explicit Carver(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t n) {
    used = (used + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += n * sizeof(T);
    return p;
  }
  size_t bytes() const { return (used + 255) & ~size_t(255); }
};

// ---- device helpers ---------------------------------------------------------
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// order-preserving map fp32 -> uint32 (larger float -> larger uint); callers
// canonicalise -0.0 to +0.0 first so that equal floats map to equal codes.
__device__ __forceinline__ uint32_t ord32(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ uint64_t ord64(double f) {
  uint64_t u = (uint64_t)__double_as_longlong(f);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ float ord32_inv(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

__device__ __forceinline__ float silu_f(float z) { return z / (1.0f + __expf(-z)); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace omni
