// Expert-parallel dispatch / combine.
#pragma once
#include <algorithm>

#include "common.cuh"

namespace omni {

constexpr int kMaxRanks = 16;

size_t ep_pack_ws_bytes(int64_t L, int R);
omnimoe_status ep_pack(int dtype, int64_t L, int d, int hk, int R, int64_t n_per, const void* x, const int32_t* idx,
                       const float* gate, void* x_send, int32_t* rec_send, int32_t* inv, int32_t* offsets,
                       int64_t* counts, void* ws, cudaStream_t st);
omnimoe_status ep_unpack(const int32_t* rec, int64_t M, int R, const int64_t* task_off, const int64_t* tok_off,
                         int32_t* ids, float* gate, int32_t* tok, cudaStream_t st);
omnimoe_status ep_combine(const void* y_ret, int bf16, const int32_t* inv, const int64_t* tok_off, int64_t L, int d,
                          int R, float* y, cudaStream_t st);
omnimoe_status ep_partials_bf16(const float* y, int64_t n, void* out, cudaStream_t st);

}  // namespace omni
