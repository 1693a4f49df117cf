#pragma once
#include <algorithm>
#include <string>

#include "common.cuh"

namespace omni {

struct SelectParams {
  int T;               // token-heads (L*h)
  int n_rows, n_cols;  // N_r, N_c
  int top_k;           // K
  int kr1, kc1;        // min(K+1, N_r), min(K+1, N_c): per-half list lengths
  int pr, pcol, pc;    // power-of-two padded sizes: rows, cols, candidates
  float cert_eps;      // > 0: flag token-heads whose K/K+1 gap <= 4*cert_eps
};

omnimoe_status select_params(const omnimoe_dims& d, int64_t T, SelectParams* p, size_t* smem);
omnimoe_status launch_select(const SelectParams& p, size_t smem, const float* logits, int32_t* idx,
                             float* gate, float* score, int32_t* flag_list, int32_t* flag_count,
                             const int32_t* list, const int32_t* list_count, cudaStream_t st);
omnimoe_status launch_canon_logits(int dtype, const void* x, const void* sub, int d, int h, int R,
                                   float* logits, int T, const int32_t* list,
                                   const int32_t* list_count, cudaStream_t st);

}  // namespace omni
