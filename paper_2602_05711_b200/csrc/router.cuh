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
  int C;               // product candidates (a*b <= K+1)
  int pkr, pkc, pkeep; // key buffer lengths: row list, column list, K+1 selected
  int group;           // threads cooperating on one token-head: 32 (warp) or 256 (CTA)
  int groups_per_cta;
  int sorted;          // 1: ids by (key desc, id asc); 0: the K selected in candidate (rank) order
  int n_heads = 1;     // h (T = L * h): the fused route's lists are per (token, head)
};

omnimoe_status select_params(const omnimoe_dims& d, int64_t T, SelectParams* p, size_t* smem);
// ablation "w/o CPR": exact top-K of T rows of N dense logits (key order)
omnimoe_status launch_dense_select(const omnimoe_dims& d, int64_t T, const float* logits, int32_t* idx, float* gate,
                                   float* score, cudaStream_t st);
// device scratch of the layer-path selection: its product-candidate table (global memory,
// read through L1 so that the shared memory holds only per-warp buffers)
size_t select_cand_ws_bytes(const omnimoe_dims& d);
struct FusedRoute;
omnimoe_status launch_select(const SelectParams& p, size_t smem, const float* logits, int32_t* idx,
                             float* gate, float* score, uint32_t* cand_ws, cudaStream_t st,
                             const FusedRoute* fused = nullptr);

// a1: exact logits RN32(x . sub) (reading Q9), [L][h*(N_r+N_c)] fp32.
size_t exact_logits_ws_bytes(const omnimoe_dims& d, int64_t L);
omnimoe_status exact_logits(const omnimoe_dims& d, int64_t L, const void* x, const void* sub, float* logits,
                            void* ws, cudaStream_t st);

// N4 (router fusion, small K): the exact-logit GEMM keeps, in its epilogue, the top kp = K+1
// half keys of every (token, half, column half of a tile) instead of writing the logits --
// fused_cand [L][2h][2][kp] (ord32(value) << 32 | ~index-in-half, 0 = empty) and, when part
// is given, fused_part [L][2h][2] = (max, sum exp(v - max)) for the halves' logsumexp.  The
// logits are still written for the fp64 fallback (sub-key rows flagged by the limb split);
// rows flagged on the token side are recomputed into `logits` by the fp64 kernel.
struct FusedRoute {
  uint64_t* cand = nullptr;
  float2* part = nullptr;
  int kp = 0;
  const int32_t* counts = nullptr;  // [2]: flagged token rows, flagged sub-key rows (device)
  const int32_t* bad_x = nullptr;   // flagged token rows (device list)
};
int fused_kp(const omnimoe_dims& d, int64_t L);  // 0: no fused path for these dims and L
size_t fused_route_bytes(const omnimoe_dims& d, int64_t L);
omnimoe_status exact_logits_fused(const omnimoe_dims& d, int64_t L, const void* x, const void* sub, float* logits,
                                  void* ws, void* fused_ws, bool want_part, FusedRoute* fr, cudaStream_t st);
// exact fp64 double-double path: mode 0 all logits, 1 tokens in list, 2 sub-key rows in list.
omnimoe_status launch_exact_dd(int dtype, const void* x, const void* sub, int d, int NC, int L,
                               float* logits, int mode, const int32_t* list, const int32_t* list_count,
                               cudaStream_t st);

}  // namespace omni
