#pragma once
#include <algorithm>

#include "common.cuh"

namespace omni {

size_t schedule_ws_bytes(int64_t M, int64_t n_loc);
// Expert Usage / Unevenness of a plan -> out[2] (device fp64)
size_t load_stats_ws_bytes();
omnimoe_status load_stats_run(const omnimoe_plan& plan, double* out, void* ws, cudaStream_t st);  // + M + 1 ints of V-order scratch
// hk = h*K: default token of task t is t / hk when token == nullptr.
omnimoe_status schedule_run(int64_t M, const int32_t* ids, const float* gate, const int32_t* token,
                            int64_t hk, const omnimoe_plan& plan, int64_t B, int64_t Tb, int64_t n_bands,
                            void* ws, cudaStream_t st);
int64_t resolve_group_size(const omnimoe_dims& d);
// token-centric ablation executor ("w/o ECS"): straight from the routing decision
omnimoe_status expert_token_run(const omnimoe_dims& dm, int64_t L, const void* x, const void* W, const void* V,
                                const int32_t* idx, const float* gate, int64_t begin, int64_t end, float* y,
                                int accumulate, cudaStream_t st);
int64_t resolve_token_blocks(const omnimoe_dims& d, int64_t L);
// SLICED pass V: n_b expert bands for n_loc local experts and n_tok tokens
int64_t resolve_v_bands(const omnimoe_dims& d, int64_t n_loc, int64_t n_tok);
// eta = M / E|E_active| under uniform routing: tasks per active expert
double expected_eta(const omnimoe_dims& d, int64_t L);
// layer_fwd runs the token-centric executor (no schedule): the "w/o ECS" ablation, or
// AUTO with the ROWS layout when expected_eta < 2 (no reuse for ECS to exploit)
bool layer_uses_token_executor(const omnimoe_dims& d, int64_t L);
// dense.cu: the routed branch as two tcgen05 GEMMs when eta is large (AUTO, ROWS, bf16, h = 1)
bool layer_uses_dense_executor(const omnimoe_dims& d, int64_t L);
size_t dense_expert_ws_bytes(const omnimoe_dims& d, int64_t L);
omnimoe_status dense_expert_run(const omnimoe_dims& d, int64_t L, const void* x, const void* W, const void* V,
                                const int32_t* idx, const float* gate, float* y_routed, void* ws, cudaStream_t st);

// V [n][d] -> [d/32][n][32] (omnimoe_pack_v)
omnimoe_status pack_v(int64_t n, int d, const void* V, void* Vs, cudaStream_t st);

size_t expert_ws_bytes(const omnimoe_dims& d, int64_t L);
int64_t bwd_ws_tasks(const omnimoe_dims& d, int64_t L);
size_t expert_bwd_ws_bytes(const omnimoe_dims& d, int64_t L);
// SLICED executor; passes: bit 0 = pass Z, bit 1 = pass V
omnimoe_status expert_sliced_run(const omnimoe_dims& dm, int64_t L, const void* x, const void* W, const void* Vs,
                                 const omnimoe_plan& plan, float* y, int accumulate, void* ws, cudaStream_t st,
                                 int passes, int act_bf16 = 0);
// N2: routed-branch backward (expert-major plan)
omnimoe_status expert_bwd_run(const omnimoe_dims& dm, int64_t L, const void* x, const void* W, const void* V,
                              const void* Ws, const omnimoe_plan& plan, const void* dy, float* dx, float* dW_act,
                              float* dV_act, float* dgate, int accumulate_dx, void* ws, cudaStream_t st);
// act_bf16 (SLICED pass V): the activations a_t enter the slice accumulation in bf16 (the
// layer, whose output is bf16; reading Q21) or fp32 (omnimoe_expert_fwd's fp32 y_routed)
omnimoe_status expert_run(const omnimoe_dims& d, int64_t L, const void* x, const void* W,
                          const void* V, const omnimoe_plan& plan, float* y, int accumulate,
                          void* ws, cudaStream_t st, int act_bf16 = 0);

}  // namespace omni
