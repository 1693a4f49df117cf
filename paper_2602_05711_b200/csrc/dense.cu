// Routed branch as two dense tcgen05 GEMMs, for η = M / |E_active| >> 1:
// when every expert is shared by a hundred tokens or more (C4: η = 164), the per-task
// L2 -> SM row traffic of the gather executors (2 x 2d bytes per task) costs more than
// computing the masked products on the tensor cores.
//   A[l][n] = g sigma((x W^T)[l][n]) for the K selected (l, n), else 0    [L][N] bf16
//             (tcgen05, K = d; the gating is the GEMM's epilogue, Z never reaches HBM:
//             a selection bitmask, its per-word prefix counts and the gates in
//             increasing-n order tell each epilogue thread which of its 32 columns to keep)
//   y_routed = A V                    [L][d] fp32      (tcgen05, K = N; V [N][d] is read in
//             place as an MN-major B operand: TMA boxes of [64 experts][64 dims])
// This is Eq.Assemble evaluated with a dense gate matrix: the same sum,
// with the non-selected terms multiplied by exact zeros.  a = g sigma(z) is rounded to
// bf16 for the second GEMM (relative 2^-9 per term).
#include "backward.cuh"
#include "gemm.cuh"
#include "schedule.cuh"

namespace omni {
namespace {

// bit (l, n) of the selection mask: one token's K distinct ids (one head)
__global__ void dense_mask_kernel(int64_t M, int k, int words, const int32_t* __restrict__ idx,
                                  uint32_t* __restrict__ mask) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = t / k;
    const int n = idx[t];
    atomicOr(&mask[l * words + (n >> 5)], 1u << (n & 31));
  }
}

// prefix[l][j] = set bits of row l in words [0, 8j): one count per 256-column GEMM tile;
// one warp per row
__global__ void dense_prefix_kernel(int64_t L, int words, const uint32_t* __restrict__ mask,
                                    int32_t* __restrict__ prefix) {
  const int lane = threadIdx.x & 31;
  const int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (l >= L) return;
  const uint4* row = reinterpret_cast<const uint4*>(mask + l * words);
  int32_t* out = prefix + l * (words / 8);
  int run = 0;
  for (int j0 = 0; j0 < words / 8; j0 += 32) {
    const int j = j0 + lane;
    int cnt = 0;
    if (j < words / 8) {
      const uint4 a = row[2 * j], b = row[2 * j + 1];
      cnt = __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(b.x) + __popc(b.y) + __popc(b.z) +
            __popc(b.w);
    }
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (j < words / 8) out[j] = run + inc - cnt;
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// gate_c[l][rank of n among row l's set bits] = g_t: the gates in increasing-n order, which
// is the order in which the GEMM epilogue meets them
__global__ void dense_gate_kernel(int64_t M, int k, int words, const int32_t* __restrict__ idx,
                                  const float* __restrict__ gate, const uint32_t* __restrict__ mask,
                                  const int32_t* __restrict__ prefix, float* __restrict__ gate_c) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = t / k;
    const int n = idx[t], w = n >> 5, j = w >> 3;
    const uint32_t* row = mask + l * words;
    int rank = prefix[l * (words / 8) + j] + __popc(row[w] & ((1u << (n & 31)) - 1u));
    for (int i = 8 * j; i < w; ++i) rank += __popc(row[i]);
    gate_c[l * k + rank] = gate[t];
  }
}

// one CTA per token row, the whole preparation in shared memory (rows of up to
// kPrepMaxWords mask words): the row's bitmask from its K ids, the per-tile prefix counts
// (one block scan), then each task's rank among the row's set bits -> gate_c.  Replaces
// the memset + global-atomic mask + prefix + rank kernels (C4 stage a6: 1.89 -> 1.84 ms).
constexpr int kPrepMaxWords = 10240;  // 40 KB of bitmask: N <= 327,680
__global__ void __launch_bounds__(256) dense_prep_kernel(int k, int words, const int32_t* __restrict__ idx,
                                                         const float* __restrict__ gate, uint32_t* __restrict__ mask,
                                                         int32_t* __restrict__ prefix, float* __restrict__ gate_c) {
  extern __shared__ uint32_t prep_sm[];
  uint32_t* bm = prep_sm;                                        // [words]
  int* tp = reinterpret_cast<int*>(prep_sm + words);             // [words / 8] tile prefix
  __shared__ int wsum[8];
  const int64_t l = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles = words / 8;
  for (int i = tid; i < words; i += 256) bm[i] = 0u;
  __syncthreads();
  const int32_t* ids = idx + l * k;
  for (int t = tid; t < k; t += 256) {
    const int n = ids[t];
    atomicOr(&bm[n >> 5], 1u << (n & 31));
  }
  __syncthreads();
  // tile counts over a contiguous range per thread, block exclusive scan
  const int per = (tiles + 255) / 256, j0 = tid * per, j1 = min(tiles, j0 + per);
  int cnt = 0;
  for (int j = j0; j < j1; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) cnt += __popc(bm[8 * j + i]);
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int run = inc - cnt;
  for (int w = 0; w < warp; ++w) run += wsum[w];
  for (int j = j0; j < j1; ++j) {
    tp[j] = run;
#pragma unroll
    for (int i = 0; i < 8; ++i) run += __popc(bm[8 * j + i]);
  }
  __syncthreads();
  uint4* mrow = reinterpret_cast<uint4*>(mask + l * words);
  for (int i = tid; i < words / 4; i += 256) mrow[i] = reinterpret_cast<const uint4*>(bm)[i];
  for (int j = tid; j < tiles; j += 256) prefix[l * tiles + j] = tp[j];
  const float* gr = gate + l * k;
  float* gcr = gate_c + l * k;
  for (int t = tid; t < k; t += 256) {
    const int n = ids[t], w = n >> 5, j = w >> 3;
    int rank = tp[j] + __popc(bm[w] & ((1u << (n & 31)) - 1u));
    for (int i = 8 * j; i < w; ++i) rank += __popc(bm[i]);
    gcr[rank] = gr[t];
  }
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
         d.n_heads == 1 && d.top_k * tuning().dense_ratio >= N &&
         expected_eta(d, L) >= 32.0 && (double)L * pad8(N) * 6.0 <= 32.0 * (1 << 30);
}

namespace {
struct DenseWs {
  uint32_t* mask;
  int32_t* prefix;
  float* gate_c;
  __nv_bfloat16* A;
  size_t bytes;
};
DenseWs carve_dense(const omnimoe_dims& d, int64_t L, void* ws) {
  const int64_t N = d.n_rows * d.n_cols, Np = pad8(N), words = pad8((N + 31) / 32);
  Carver c(ws);
  DenseWs w;
  w.mask = c.take<uint32_t>((size_t)L * words);
  w.prefix = c.take<int32_t>((size_t)L * words / 8);
  w.gate_c = c.take<float>((size_t)L * d.top_k);
  w.A = c.take<__nv_bfloat16>((size_t)L * Np);
  w.bytes = c.bytes();
  return w;
}
}  // namespace

size_t dense_expert_ws_bytes(const omnimoe_dims& d, int64_t L) { return carve_dense(d, L, nullptr).bytes; }

omnimoe_status dense_expert_run(const omnimoe_dims& d, int64_t L, const void* x, const void* W, const void* V,
                                const int32_t* idx, const float* gate, float* y_routed, void* ws, cudaStream_t st) {
  const int64_t N = d.n_rows * d.n_cols, Np = pad8(N), M = L * d.n_heads * d.top_k;
  const int words = (int)pad8((N + 31) / 32), k = (int)(d.n_heads * d.top_k);
  DenseWs w = carve_dense(d, L, ws);
  if (M > 0 && words <= kPrepMaxWords) {
    const size_t sm = (size_t)words * 4 + (size_t)(words / 8) * 4;  // <= 45 KB: no opt-in needed
    dense_prep_kernel<<<(unsigned)L, 256, sm, st>>>(k, words, idx, gate, w.mask, w.prefix, w.gate_c);
    OMNI_CHECK_LAUNCH("dense_prep_kernel");
  } else if (M > 0) {  // very wide rows: global-memory bitmask
    if (cudaMemsetAsync(w.mask, 0, (size_t)L * words * 4, st) != cudaSuccess) {
      set_error("dense executor: memset failed");
      return OMNIMOE_ERR_CUDA;
    }
    dense_mask_kernel<<<num_sms() * 8, 256, 0, st>>>(M, k, words, idx, w.mask);
    OMNI_CHECK_LAUNCH("dense_mask_kernel");
    dense_prefix_kernel<<<(unsigned)((L * 32 + 255) / 256), 256, 0, st>>>(L, words, w.mask, w.prefix);
    OMNI_CHECK_LAUNCH("dense_prefix_kernel");
    dense_gate_kernel<<<num_sms() * 8, 256, 0, st>>>(M, k, words, idx, gate, w.mask, w.prefix, w.gate_c);
    OMNI_CHECK_LAUNCH("dense_gate_kernel");
  }
  GemmArgs g1;  // A = mask (.) g act(x W^T), written once in bf16 by the GEMM epilogue
  g1.M = (int)L;
  g1.N = (int)N;
  g1.K = (int)d.d;
  g1.out = w.A;
  g1.mask = w.mask;
  g1.mask_prefix = w.prefix;
  g1.gate_c = w.gate_c;
  g1.mask_words = words;
  g1.gate_ld = k;
  g1.out_ld = (int)Np;
  g1.act = d.act;
  OMNI_TRY(gemm_bf16(EPI_GATED, x, W, g1, st));
  GemmArgs g2;  // y_routed = A V, V read in place as an MN-major operand (rows >= N: zeros)
  g2.M = (int)L;
  g2.N = (int)d.d;
  g2.K = (int)Np;
  g2.b_mn = 1;
  g2.b_rows = N;
  g2.out_f32 = y_routed;
  return gemm_bf16(EPI_F32, w.A, V, g2, st);
}

}  // namespace omni
