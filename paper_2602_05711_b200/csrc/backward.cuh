#pragma once
#include <algorithm>

#include "common.cuh"

namespace omni {

inline int64_t pad8(int64_t n) { return (n + 7) / 8 * 8; }
// out[c][r] = in[r][c] for 2-byte elements; out row stride ld (0: R), columns [R, ld) zeroed
omnimoe_status transpose16(const void* in, void* out, int64_t R, int64_t C, cudaStream_t st, int64_t ld = 0);

// N2: router-gate and shared-MLP backward (backward.cu)
size_t router_bwd_ws_bytes(const omnimoe_dims& d, int64_t L);
size_t mlp_bwd_ws_bytes(const omnimoe_dims& d, int64_t L);
omnimoe_status router_bwd_run(const omnimoe_dims& d, int64_t L, const void* x, const void* sub, const int32_t* idx,
                              const float* gate, const float* dgate, float* dx, int accumulate_dx, float* dsub,
                              void* ws, cudaStream_t st);
omnimoe_status mlp_bwd_run(const omnimoe_dims& d, int64_t L, const void* x, const void* wgu, const void* wdn,
                           const void* dy, float* dx, int accumulate_dx, float* dwgu, float* dwdn, void* ws,
                           cudaStream_t st);

}  // namespace omni
