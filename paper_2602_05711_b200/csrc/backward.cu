// N2: backward of the router gates and of the shared dense MLP.
// (The routed branch's backward, expert_bwd_kernel, lives in expert.cu next to the
// forward executors it mirrors.)  Every contraction runs on the tcgen05 GEMM engine
// (gemm.cu, C = A . B^T with K-major bf16 operands); the operands it needs in the
// other orientation are produced by a tiled bf16 transpose.
//
//  router:  dkappa_k = g_k (dgate_k - sum_j g_j dgate_j) over the K selected keys of
//           a token-head (Eq.Gate); ds_r[i] += dkappa, ds_c[j] +=
//           dkappa for the selected cell (i, j) (Eq.S); then
//           dsub = ds^T x and dx += ds sub (Eq.Logits).
//  MLP:     G|U = x W_gu^T, dH = dy W_down, H = SiLU(G) U, dU = dH SiLU(G),
//           dG = dH U SiLU'(G); dW_down = dy^T H, dW_gu = [dG|dU]^T x,
//           dx += [dG|dU] W_gu  (reading Q2).
#include "backward.cuh"
#include "gemm.cuh"

namespace omni {

// out[c][r] = in[r][c] for 2-byte elements (out row stride ld >= R, columns r in [R, ld)
// zero-filled so that the GEMM's K = ld stays a multiple of 8), 32 x 32 tiles in smem
namespace {
__global__ void __launch_bounds__(256) transpose16_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out,
                                                          int64_t R, int64_t C, int64_t ld) {
  __shared__ uint16_t tile[32][33];
  const int64_t nty = (ld + 31) / 32, ntx = (C + 31) / 32;
  for (int64_t t = blockIdx.x; t < nty * ntx; t += gridDim.x) {
    const int64_t r0 = (t / ntx) * 32, c0 = (t % ntx) * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int64_t r = r0 + i, c = c0 + threadIdx.x;
      tile[i][threadIdx.x] = (r < R && c < C) ? in[r * C + c] : 0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
      const int64_t c = c0 + i, r = r0 + threadIdx.x;
      if (c < C && r < ld) out[c * ld + r] = tile[threadIdx.x][i];
    }
    __syncthreads();
  }
}

}  // namespace

omnimoe_status transpose16(const void* in, void* out, int64_t R, int64_t C, cudaStream_t st, int64_t ld) {
  if (ld == 0) ld = R;
  if (R == 0 || C == 0) return OMNIMOE_OK;
  const int64_t tiles = ((ld + 31) / 32) * ((C + 31) / 32);
  transpose16_kernel<<<(int)std::min<int64_t>(tiles, num_sms() * 16), dim3(32, 8), 0, st>>>(
      static_cast<const uint16_t*>(in), static_cast<uint16_t*>(out), R, C, ld);
  OMNI_CHECK_LAUNCH("transpose16_kernel");
  return OMNIMOE_OK;
}


namespace {

__global__ void add_f32_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

omnimoe_status add_f32(float* dst, const float* src, int64_t n, int accumulate, cudaStream_t st) {
  if (!accumulate) {
    if (cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      set_error("backward: copy failed");
      return OMNIMOE_ERR_CUDA;
    }
    return OMNIMOE_OK;
  }
  add_f32_kernel<<<num_sms() * 4, 256, 0, st>>>(dst, src, n);
  OMNI_CHECK_LAUNCH("add_f32_kernel");
  return OMNIMOE_OK;
}

// one warp per token-head: dkappa over the K selected keys, scattered into the
// token-head's ds row (shared memory, lane 0 in k order: deterministic), written as a
// bf16 pair hi + lo (ds2[t][r] = hi, ds2[t][R_all + r] = lo = bf16(ds - hi)) so that
// the GEMMs see ~16 significant bits: the rows of ds sum to zero over a token-head,
// and a single bf16 rounding loses too much to that cancellation
__global__ void __launch_bounds__(256)
    router_ds_kernel(int64_t T, int R, int Nr, int Nc, int K, const int32_t* __restrict__ idx,
                     const float* __restrict__ gate, const float* __restrict__ dgate, __nv_bfloat16* __restrict__ ds,
                     int64_t hR, int h) {
  extern __shared__ float rows[];  // [8 warps][R]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* row = rows + (size_t)w * R;
  const int64_t gw = blockIdx.x * 8 + w, nw = (int64_t)gridDim.x * 8;
  for (int64_t t = gw; t < T; t += nw) {
    float dot = 0.f;
    for (int k = lane; k < K; k += 32) dot += gate[t * K + k] * dgate[t * K + k];
    dot = warp_sum(dot);
    for (int r = lane; r < R; r += 32) row[r] = 0.f;
    __syncwarp();
    if (lane == 0)
      for (int k = 0; k < K; ++k) {
        const float dk = gate[t * K + k] * (dgate[t * K + k] - dot);
        const int n = idx[t * K + k];
        row[n / Nc] += dk;
        row[Nr + n % Nc] += dk;
      }
    __syncwarp();
    const int64_t l = t / h, base = l * 2 * hR + (t - l * h) * R;
    for (int r = lane; r < R; r += 32) {
      const __nv_bfloat16 hi = __float2bfloat16_rn(row[r]);
      ds[base + r] = hi;
      ds[base + hR + r] = __float2bfloat16_rn(row[r] - __bfloat162float(hi));
    }
    __syncwarp();
  }
}

// from G|U (fp32 [L][2F]) and dH (fp32 [L][F]): H as a bf16 pair (H2 [L][hi F | lo F])
// and dG|dU as a bf16 pair (dgu2 [L][dG_hi dU_hi | dG_lo dU_lo], 4F): hi = bf16(v),
// lo = bf16(v - hi), ~16 significant bits for the GEMMs that contract them
__global__ void swiglu_bwd_kernel(const float* __restrict__ gu, const float* __restrict__ dh, int64_t L, int F,
                                  __nv_bfloat16* __restrict__ H2, __nv_bfloat16* __restrict__ dgu2) {
  const int64_t n = L * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / F;
    const int f = (int)(i - l * F);
    const float g = gu[l * 2 * F + f], u = gu[l * 2 * F + F + f], d = dh[i];
    const float sg = 1.0f / (1.0f + __expf(-g));
    const float silu = g * sg, dsilu = sg * (1.0f + g * (1.0f - sg));
    const float h = silu * u, dg = d * u * dsilu, du = d * silu;
    const __nv_bfloat16 hh = __float2bfloat16_rn(h), gh = __float2bfloat16_rn(dg), uh = __float2bfloat16_rn(du);
    H2[l * 2 * F + f] = hh;
    H2[l * 2 * F + F + f] = __float2bfloat16_rn(h - __bfloat162float(hh));
    dgu2[l * 4 * F + f] = gh;
    dgu2[l * 4 * F + F + f] = uh;
    dgu2[l * 4 * F + 2 * F + f] = __float2bfloat16_rn(dg - __bfloat162float(gh));
    dgu2[l * 4 * F + 3 * F + f] = __float2bfloat16_rn(du - __bfloat162float(uh));
  }
}

omnimoe_status gemm_f32out(const void* A, const void* B, int64_t M, int64_t N, int64_t K, float* C, cudaStream_t st) {
  GemmArgs g;
  g.M = (int)M;
  g.N = (int)N;
  g.K = (int)K;
  g.out_f32 = C;
  return gemm_bf16(EPI_F32, A, B, g, st);
}

struct RouterBwdWs {
  __nv_bfloat16 *ds, *dsT, *sub2, *subT, *xT;
  float* tmp;
};
size_t router_bwd_carve(const omnimoe_dims& d, int64_t L, void* ws, RouterBwdWs* o) {
  Carver c(ws);
  const int64_t hR = d.n_heads * (d.n_rows + d.n_cols);
  auto ds = c.take<__nv_bfloat16>((size_t)L * 2 * hR);   // [L][hi | lo]
  auto dsT = c.take<__nv_bfloat16>((size_t)pad8(L) * 2 * hR);  // [hi^T ; lo^T], rows of pad8(L)
  auto sub2 = c.take<__nv_bfloat16>((size_t)hR * 2 * d.d); // [sub ; sub]
  auto subT = c.take<__nv_bfloat16>((size_t)hR * 2 * d.d); // [d][sub^T | sub^T]
  auto xT = c.take<__nv_bfloat16>((size_t)pad8(L) * d.d);
  auto tmp = c.take<float>((size_t)std::max<int64_t>(L, hR) * d.d);
  if (o) *o = RouterBwdWs{ds, dsT, sub2, subT, xT, tmp};
  return c.bytes();
}

struct MlpBwdWs {
  float *gu, *dh, *tmp;
  __nv_bfloat16 *H2, *dgu2, *wdT, *wgu2, *wguT, *dyT, *HT, *dguT, *xT;
};
size_t mlp_bwd_carve(const omnimoe_dims& d, int64_t L, void* ws, MlpBwdWs* o) {
  Carver c(ws);
  const int64_t F = d.d_ff, D = d.d, Lp = pad8(L);
  MlpBwdWs w;
  w.gu = c.take<float>((size_t)L * 2 * F);
  w.dh = c.take<float>((size_t)L * F);
  w.tmp = c.take<float>((size_t)std::max<int64_t>(L * D, 2 * F * D));
  w.H2 = c.take<__nv_bfloat16>((size_t)L * 2 * F);
  w.dgu2 = c.take<__nv_bfloat16>((size_t)L * 4 * F);
  w.wdT = c.take<__nv_bfloat16>((size_t)F * D);
  w.wgu2 = c.take<__nv_bfloat16>((size_t)4 * F * D);
  w.wguT = c.take<__nv_bfloat16>((size_t)4 * F * D);
  w.dyT = c.take<__nv_bfloat16>((size_t)Lp * D);
  w.HT = c.take<__nv_bfloat16>((size_t)Lp * 2 * F);
  w.dguT = c.take<__nv_bfloat16>((size_t)Lp * 4 * F);
  w.xT = c.take<__nv_bfloat16>((size_t)Lp * D);
  if (o) *o = w;
  return c.bytes();
}

}  // namespace

size_t router_bwd_ws_bytes(const omnimoe_dims& d, int64_t L) { return router_bwd_carve(d, L, nullptr, nullptr); }
size_t mlp_bwd_ws_bytes(const omnimoe_dims& d, int64_t L) { return mlp_bwd_carve(d, L, nullptr, nullptr); }

omnimoe_status router_bwd_run(const omnimoe_dims& d, int64_t L, const void* x, const void* sub, const int32_t* idx,
                              const float* gate, const float* dgate, float* dx, int accumulate_dx, float* dsub,
                              void* ws, cudaStream_t st) {
  RouterBwdWs w;
  router_bwd_carve(d, L, ws, &w);
  const int R = (int)(d.n_rows + d.n_cols);
  const int64_t hR = d.n_heads * R, T = L * d.n_heads;
  const size_t smem = (size_t)8 * R * sizeof(float);
  if (smem > 200 * 1024) {
    set_error("router_bwd: N_r + N_c too large for the per-warp ds rows");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (cudaFuncSetAttribute(router_ds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("router_bwd: cannot set shared memory");
    return OMNIMOE_ERR_CUDA;
  }
  router_ds_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((T + 7) / 8, num_sms() * 2)), 256, smem, st>>>(
      T, R, (int)d.n_rows, (int)d.n_cols, (int)d.top_k, idx, gate, dgate, w.ds, hR, (int)d.n_heads);
  OMNI_CHECK_LAUNCH("router_ds_kernel");
  // dsub [hR][d] = hi^T x + lo^T x :  A = [hi^T ; lo^T] halves [hR][L], B = x^T [d][L]
  const int64_t Lp = pad8(L);
  OMNI_TRY(transpose16(w.ds, w.dsT, L, 2 * hR, st, Lp));
  OMNI_TRY(transpose16(x, w.xT, L, d.d, st, Lp));
  OMNI_TRY(gemm_f32out(w.dsT, w.xT, hR, d.d, Lp, dsub, st));
  OMNI_TRY(gemm_f32out(w.dsT + (size_t)hR * Lp, w.xT, hR, d.d, Lp, w.tmp, st));
  OMNI_TRY(add_f32(dsub, w.tmp, hR * d.d, 1, st));
  // dx += [hi | lo] [sub ; sub] :  A = ds2 [L][2hR], B = [sub^T | sub^T] [d][2hR]
  const size_t sub_bytes = (size_t)hR * d.d * 2;
  if (cudaMemcpyAsync(w.sub2, sub, sub_bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(reinterpret_cast<char*>(w.sub2) + sub_bytes, sub, sub_bytes, cudaMemcpyDeviceToDevice, st) !=
          cudaSuccess) {
    set_error("router_bwd: copy failed");
    return OMNIMOE_ERR_CUDA;
  }
  OMNI_TRY(transpose16(w.sub2, w.subT, 2 * hR, d.d, st));
  OMNI_TRY(gemm_f32out(w.ds, w.subT, L, d.d, 2 * hR, w.tmp, st));
  return add_f32(dx, w.tmp, L * d.d, accumulate_dx, st);
}

omnimoe_status mlp_bwd_run(const omnimoe_dims& d, int64_t L, const void* x, const void* wgu, const void* wdn,
                           const void* dy, float* dx, int accumulate_dx, float* dwgu, float* dwdn, void* ws,
                           cudaStream_t st) {
  MlpBwdWs w;
  mlp_bwd_carve(d, L, ws, &w);
  const int64_t F = d.d_ff, D = d.d, Lp = pad8(L);  // Lp: K of the token-contracted GEMMs, zero-padded
  OMNI_TRY(gemm_f32out(x, wgu, L, 2 * F, D, w.gu, st));       // G|U = x W_gu^T
  OMNI_TRY(transpose16(wdn, w.wdT, D, F, st));                 // W_down^T [F][D]
  OMNI_TRY(gemm_f32out(dy, w.wdT, L, F, D, w.dh, st));        // dH = dy W_down
  swiglu_bwd_kernel<<<num_sms() * 8, 256, 0, st>>>(w.gu, w.dh, L, (int)F, w.H2, w.dgu2);
  OMNI_CHECK_LAUNCH("swiglu_bwd_kernel");
  // dW_down = dy^T (H_hi + H_lo)
  OMNI_TRY(transpose16(dy, w.dyT, L, D, st, Lp));
  OMNI_TRY(transpose16(w.H2, w.HT, L, 2 * F, st, Lp));
  OMNI_TRY(gemm_f32out(w.dyT, w.HT, D, F, Lp, dwdn, st));
  OMNI_TRY(gemm_f32out(w.dyT, w.HT + (size_t)F * Lp, D, F, Lp, w.tmp, st));
  OMNI_TRY(add_f32(dwdn, w.tmp, D * F, 1, st));
  // dW_gu = (dGU_hi + dGU_lo)^T x
  OMNI_TRY(transpose16(w.dgu2, w.dguT, L, 4 * F, st, Lp));
  OMNI_TRY(transpose16(x, w.xT, L, D, st, Lp));
  OMNI_TRY(gemm_f32out(w.dguT, w.xT, 2 * F, D, Lp, dwgu, st));
  OMNI_TRY(gemm_f32out(w.dguT + (size_t)2 * F * Lp, w.xT, 2 * F, D, Lp, w.tmp, st));
  OMNI_TRY(add_f32(dwgu, w.tmp, 2 * F * D, 1, st));
  // dx += [dGU_hi | dGU_lo] [W_gu ; W_gu]
  const size_t wb = (size_t)2 * F * D * 2;
  if (cudaMemcpyAsync(w.wgu2, wgu, wb, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(reinterpret_cast<char*>(w.wgu2) + wb, wgu, wb, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
    set_error("shared_mlp_bwd: copy failed");
    return OMNIMOE_ERR_CUDA;
  }
  OMNI_TRY(transpose16(w.wgu2, w.wguT, 4 * F, D, st));          // [D][4F]
  OMNI_TRY(gemm_f32out(w.dgu2, w.wguT, L, D, 4 * F, w.tmp, st));
  return add_f32(dx, w.tmp, L * D, accumulate_dx, st);
}

}  // namespace omni
