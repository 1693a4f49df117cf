// Routed branch as two dense tcgen05 GEMMs, for η = M / |E_active| >> 1:
// when every expert is shared by a hundred tokens or more (C4: η = 164), the per-task
// L2 -> SM row traffic of the gather executors (2 x 2d bytes per task) costs more than
// computing the masked products on the tensor cores.
//   Z = x W^T                         [L][N] fp32      (tcgen05, K = d)
//   A[l][n] = g sigma(Z[l][n]) for the K selected (l, n), else 0   [L][N] bf16
//   y_routed = A V                    [L][d] fp32      (tcgen05, K = N, V transposed)
// This is Eq.Assemble evaluated with a dense gate matrix: the same sum,
// with the non-selected terms multiplied by exact zeros.  a = g sigma(z) is rounded to
// bf16 for the second GEMM (relative 2^-9 per term).
#include "backward.cuh"
#include "gemm.cuh"
#include "schedule.cuh"

namespace omni {
namespace {

__global__ void dense_act_kernel(int64_t M, int hk, int64_t N, int64_t Np, const int32_t* __restrict__ idx,
                                 const float* __restrict__ gate, const float* __restrict__ Z,
                                 __nv_bfloat16* __restrict__ A, int act) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = t / hk, n = idx[t];
    const float z = Z[l * N + n];
    A[l * Np + n] = __float2bfloat16_rn(gate[t] * (act == OMNIMOE_IDENTITY ? z : silu_f(z)));
  }
}

int env_int_d(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

}  // namespace

bool layer_uses_dense_executor(const omnimoe_dims& d, int64_t L) {
  const int64_t N = d.n_rows * d.n_cols;
  // Dense work is 4 L N d FLOPs on ~1.2 PF/s of tensor cores; the gather executors move
  // 4 d bytes per task (L K tasks) at ~12 TB/s from L2: dense wins once K / N exceeds
  // ~1% (measured: C4 and C4' at K/N = 4%: 4.2 vs 7.0 ms and 1.9 vs 2.8 ms; C4'' at
  // 0.5%: 2.9 vs 1.4 ms), so the rule asks for K >= N / 40 and eta >= 32 (every expert
  // shared by many tokens).  One head: a token's K ids are distinct, A needs no sums.
  return d.expert_kernel == OMNIMOE_EXPERT_AUTO && d.v_layout == OMNIMOE_V_ROWS && d.dtype == OMNIMOE_BF16 &&
         d.n_heads == 1 && d.top_k * env_int_d("OMNIMOE_DENSE_RATIO", 40) >= N &&
         expected_eta(d, L) >= 32.0 && (double)L * pad8(N) * 6.0 <= 32.0 * (1 << 30);
}

size_t dense_expert_ws_bytes(const omnimoe_dims& d, int64_t L) {
  const int64_t N = d.n_rows * d.n_cols, Np = pad8(N);
  Carver c(nullptr);
  c.take<float>((size_t)L * N);               // Z
  c.take<__nv_bfloat16>((size_t)L * Np);      // A
  c.take<__nv_bfloat16>((size_t)d.d * Np);    // V^T
  return c.bytes();
}

omnimoe_status dense_expert_run(const omnimoe_dims& d, int64_t L, const void* x, const void* W, const void* V,
                                const int32_t* idx, const float* gate, float* y_routed, void* ws, cudaStream_t st) {
  const int64_t N = d.n_rows * d.n_cols, Np = pad8(N), M = L * d.n_heads * d.top_k;
  Carver c(ws);
  float* Z = c.take<float>((size_t)L * N);
  auto A = c.take<__nv_bfloat16>((size_t)L * Np);
  auto VT = c.take<__nv_bfloat16>((size_t)d.d * Np);
  GemmArgs g1;
  g1.M = (int)L;
  g1.N = (int)N;
  g1.K = (int)d.d;
  g1.out_f32 = Z;
  OMNI_TRY(gemm_bf16(EPI_F32, x, W, g1, st));  // Z = x W^T
  if (cudaMemsetAsync(A, 0, (size_t)L * Np * 2, st) != cudaSuccess) {
    set_error("dense executor: memset failed");
    return OMNIMOE_ERR_CUDA;
  }
  dense_act_kernel<<<kSMs * 8, 256, 0, st>>>(M, (int)(d.n_heads * d.top_k), N, Np, idx, gate, Z, A, d.act);
  OMNI_CHECK_LAUNCH("dense_act_kernel");
  OMNI_TRY(transpose16(V, VT, N, d.d, st, Np));  // V^T [d][Np], zero-padded
  GemmArgs g2;
  g2.M = (int)L;
  g2.N = (int)d.d;
  g2.K = (int)Np;
  g2.out_f32 = y_routed;
  return gemm_bf16(EPI_F32, A, VT, g2, st);  // y_routed = A V
}

}  // namespace omni
