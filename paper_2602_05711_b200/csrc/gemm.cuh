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
  EPI_GATED = 3,   // out[m][n] = bf16(g_mn act(acc)) where mask bit (m,n) is set, else 0
                   // (dense routed branch): g_mn = gate_c[m][rank of n in row m]
};

struct GemmArgs {
  int M = 0, N = 0, K = 0;        // N: output columns (for SWIGLU: d_ff)
  float* out_f32 = nullptr;       // EPI_F32
  void* out = nullptr;            // EPI_SWIGLU / EPI_ADD output (bf16 or fp32 by dtype)
  const float* addend = nullptr;  // EPI_ADD (nullable)
  // EPI_GATED: mask [M][mask_words] bit n%32 of word n/32 (mask_words % 8 == 0);
  // mask_prefix[m][j] = set bits of row m in words [0, 8j) (one count per 256-column tile);
  // gate_c [M][gate_ld] gates in increasing-n order; out bf16 [M][out_ld] (columns
  // [N, out_ld) written as zeros).
  const uint32_t* mask = nullptr;
  const int32_t* mask_prefix = nullptr;
  const float* gate_c = nullptr;
  int mask_words = 0, gate_ld = 0, out_ld = 0, act = 0;
  // tile order: -1 = auto (m fastest when A is small enough to stay L2-resident while B
  // streams once), 0 = n fastest, 1 = m fastest
  int m_fast = -1;
  // B given MN-major: B is [K][N] row-major (b_rows rows; rows [b_rows, K) read as zeros),
  // i.e. C = A . B instead of A . B^T -- no transposed copy (EPI_F32 only)
  int b_mn = 0;
  int64_t b_rows = 0;
  // EPI_SWIGLU: write H as a bf16 pair, row m = [hi (N) | lo (N)], hi = bf16(h), lo = bf16(h - hi)
  // (~16 significant bits for the GEMM that contracts it; out row stride 2N)
  int h_split = 0;
  // B's K extent when smaller than A's: K block kb of A meets K block kb mod (b_kwrap / 64) of B
  // (C = [H_hi | H_lo] . [B | B]^T without a duplicated B); b_kwrap % 64 == 0, K % b_kwrap == 0
  int b_kwrap = 0;
};

// bf16 operands.  For EPI_SWIGLU, B is w_gate_up [2N][K]: gate rows [0,N), up rows [N,2N).
omnimoe_status gemm_bf16(int epi, const void* A, const void* B, const GemmArgs& a,
                         cudaStream_t st);
// fp32 operands (OMNIMOE_F32 mode), same semantics, fp32 outputs.
omnimoe_status gemm_f32(int epi, const float* A, const float* B, const GemmArgs& a,
                        cudaStream_t st);

}  // namespace omni
