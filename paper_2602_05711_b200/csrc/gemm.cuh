// GEMM engine interface: C = A . B^T with A [M][K], B [N][K] (both K-major).
// bf16 path: hand-written tcgen05 kernel (TMA -> SMEM ring -> tcgen05.mma ->
// TMEM -> fused epilogue).  fp32 path (correctness mode): SIMT FFMA kernel.
#pragma once
#include "common.cuh"

namespace omni {

enum GemmEpi {
  EPI_F32 = 0,     // out_f32[m][n] = acc                      (router logits, a1)
  EPI_SWIGLU = 1,  // out[m][f] = silu(acc_gate) * acc_up      (shared MLP GEMM-1, a7)
  EPI_ADD = 2,     // out[m][n] = acc + addend[m][n]           (shared MLP GEMM-2 + combine, a7/a8)
};

struct GemmArgs {
  int M = 0, N = 0, K = 0;        // N: output columns (for SWIGLU: d_ff)
  float* out_f32 = nullptr;       // EPI_F32
  void* out = nullptr;            // EPI_SWIGLU / EPI_ADD output (bf16 or fp32 by dtype)
  const float* addend = nullptr;  // EPI_ADD (nullable)
};

// bf16 operands.  For EPI_SWIGLU, B is w_gate_up [2N][K]: gate rows [0,N), up rows [N,2N).
omnimoe_status gemm_bf16(int epi, const void* A, const void* B, const GemmArgs& a,
                         cudaStream_t st);
// fp32 operands (OMNIMOE_F32 mode), same semantics, fp32 outputs.
omnimoe_status gemm_f32(int epi, const float* A, const float* B, const GemmArgs& a,
                        cudaStream_t st);

}  // namespace omni
