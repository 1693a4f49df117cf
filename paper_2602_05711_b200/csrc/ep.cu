// Expert-parallel dispatch / combine kernels.
//
// Rank r owns the flat expert ids [r*n_per, (r+1)*n_per) -- whole grid rows,
// because n = i*N_c + j (reading Q6) -- and L_loc of the tokens.  After routing
// its tokens (ids are bit-identical to a single-GPU run: routing is per token),
// a rank sends every destination s
//   * each of its tokens that has >= 1 task on s, ONCE (x row, "slot" = its
//     position in the message to s, tokens ascending), and
//   * one record per task on s: (local expert id, gate bits, slot).
// The receiver turns records into a task list over "virtual tokens" (the
// received x rows) and runs the local schedule + expert_fwd; partial y rows go
// back in the same slot layout and the home rank adds them, rank by rank in a
// fixed order (no atomics: deterministic), before the shared MLP + combine.
//
//  ep_count_kernel    per token: tasks per destination -> cnt[s][l], has[s][l]
//  (scan)             s-major exclusive scans -> task and token offsets
//  ep_pack_kernel     per token (one warp): x rows to x_send, records to rec_send,
//                     inv[s][l] = slot of token l in the message to s (or -1)
//  ep_unpack_kernel   records -> (local id, gate, virtual token) task arrays
//  ep_partials_kernel the partial rows of a shard, fp32 -> bf16 for the return trip
//  ep_combine_kernel  y_routed[l] = sum over s = 0..R-1 of y_ret[s][inv[s][l]]
#include "ep.cuh"

namespace omni {
namespace {

__global__ void ep_count_kernel(const int32_t* __restrict__ idx, int64_t L, int hk, int R, int64_t n_per,
                                int32_t* __restrict__ cnt, int32_t* __restrict__ has) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L; l += (int64_t)gridDim.x * blockDim.x) {
    int c[kMaxRanks];
#pragma unroll
    for (int s = 0; s < kMaxRanks; ++s) c[s] = 0;
    for (int k = 0; k < hk; ++k) {
      const int s = (int)(idx[l * hk + k] / n_per);
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q) c[q] += (q == s);
    }
    for (int s = 0; s < R; ++s) {
      cnt[(int64_t)s * L + l] = c[s];
      has[(int64_t)s * L + l] = c[s] > 0;
    }
  }
}

// exclusive scan of an int32 array (single CTA, chunked) -- sizes here are R*L_loc
__global__ void __launch_bounds__(1024) ep_scan_kernel(const int32_t* __restrict__ in, int64_t n,
                                                       int32_t* __restrict__ out) {
  __shared__ int ws[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t b = 0; b < n; b += 1024) {
    const int64_t i = b + threadIdx.x;
    const int v = i < n ? in[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    int wp = 0, tot = 0;
    for (int q = 0; q < 32; ++q) {
      if (q < w) wp += ws[q];
      tot += ws[q];
    }
    if (i < n) out[i] = carry + wp + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

template <typename T>
__global__ void ep_pack_kernel(const T* __restrict__ x, const int32_t* __restrict__ idx, const float* __restrict__ gate,
                               int64_t L, int d, int hk, int R, int64_t n_per, const int32_t* __restrict__ task_pos,
                               const int32_t* __restrict__ tok_pos, T* __restrict__ x_send,
                               int32_t* __restrict__ rec_send, int32_t* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int vec = 16 / (int)sizeof(T);
  for (int64_t l = gw; l < L; l += nw) {
    for (int s = 0; s < R; ++s) {
      const int64_t sl = (int64_t)s * L + l;
      const int has = tok_pos[sl + 1] - tok_pos[sl];
      if (!has) {
        if (lane == 0) inv[sl] = -1;
        continue;
      }
      const int64_t pos = tok_pos[sl];  // row in the concatenated send buffer
      const int slot = (int)(pos - tok_pos[(int64_t)s * L]);
      if (lane == 0) inv[sl] = slot;
      const uint4* src = reinterpret_cast<const uint4*>(x + l * d);
      uint4* dst = reinterpret_cast<uint4*>(x_send + pos * d);
      for (int c = lane; c < d / vec; c += 32) dst[c] = src[c];
    }
    // records of this token's tasks, in task order per destination: 32 tasks at
    // a time, rank among same-destination lanes by __match_any_sync
    int base = lane < R ? task_pos[(int64_t)lane * L + l] : 0;  // lane s: next record slot of dest s
    const int slot_s = lane < R ? (int)(tok_pos[(int64_t)lane * L + l] - tok_pos[(int64_t)lane * L]) : 0;
    for (int k0 = 0; k0 < hk; k0 += 32) {
      const int k = k0 + lane;
      const bool ok = k < hk;
      const int32_t n = ok ? idx[l * hk + k] : 0;
      const int s = ok ? (int)(n / n_per) : kMaxRanks;
      const unsigned peers = __match_any_sync(0xffffffffu, s);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      const int b = __shfl_sync(0xffffffffu, base, s & 31);
      const int sl = __shfl_sync(0xffffffffu, slot_s, s & 31);
      if (ok) {
        const int64_t p = (int64_t)b + rank;
        rec_send[3 * p] = (int32_t)(n - (int64_t)s * n_per);
        rec_send[3 * p + 1] = __float_as_int(gate[l * hk + k]);
        rec_send[3 * p + 2] = sl;
      }
      // advance each destination's counter by its count in this chunk
      int add = 0;
      for (int q = 0; q < R; ++q) {
        const unsigned m = __ballot_sync(0xffffffffu, ok && s == q);
        if (lane == q) add = __popc(m);
      }
      base += add;
    }
  }
}

__global__ void ep_offsets_kernel(const int32_t* __restrict__ tok_pos, const int32_t* __restrict__ task_pos,
                                  int64_t L, int R, int32_t* __restrict__ offsets, int64_t* __restrict__ counts) {
  const int s = threadIdx.x;
  if (s <= R) {
    offsets[s] = tok_pos[(int64_t)s * L];
    offsets[R + 1 + s] = task_pos[(int64_t)s * L];
  }
  if (counts && s < R) {  // (rows, records) per destination: the all-to-all split sizes
    counts[2 * s] = tok_pos[(int64_t)(s + 1) * L] - tok_pos[(int64_t)s * L];
    counts[2 * s + 1] = task_pos[(int64_t)(s + 1) * L] - task_pos[(int64_t)s * L];
  }
}

__global__ void ep_unpack_kernel(const int32_t* __restrict__ rec, int64_t M, int R,
                                 const int64_t* __restrict__ task_off, const int64_t* __restrict__ tok_off,
                                 int32_t* __restrict__ ids, float* __restrict__ gate, int32_t* __restrict__ tok) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += (int64_t)gridDim.x * blockDim.x) {
    int src = 0;
    while (src + 1 < R && task_off[src + 1] <= t) ++src;
    ids[t] = rec[3 * t];
    gate[t] = __int_as_float(rec[3 * t + 1]);
    tok[t] = (int32_t)(tok_off[src] + rec[3 * t + 2]);
  }
}

template <bool BF16>
__global__ void ep_combine_kernel(const void* __restrict__ y_ret, const int32_t* __restrict__ inv,
                                  const int64_t* __restrict__ tok_off, int64_t L, int d, int R,
                                  float* __restrict__ y) {
  const int64_t n4 = (int64_t)L * d / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = (i * 4) / d;
    const int c = (int)((i * 4) % d);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < R; ++s) {  // fixed rank order
      const int slot = inv[(int64_t)s * L + l];
      if (slot < 0) continue;
      float4 v;
      if (BF16) {
        const uint2 u = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(y_ret) + (tok_off[s] + slot) * d + c);
        v = make_float4(bf16_lo(u.x), bf16_hi(u.x), bf16_lo(u.y), bf16_hi(u.y));
      } else {
        v = *reinterpret_cast<const float4*>(static_cast<const float*>(y_ret) + (tok_off[s] + slot) * d + c);
      }
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(y)[i] = acc;
  }
}

__global__ void ep_partials_kernel(const float4* __restrict__ y, int64_t n4, uint2* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = y[i];
    out[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
}

int grid_of(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, num_sms() * 16));
}

}  // namespace

size_t ep_pack_ws_bytes(int64_t L, int R) {
  Carver c(nullptr);
  c.take<int32_t>((size_t)R * L);      // cnt
  c.take<int32_t>((size_t)R * L);      // has
  c.take<int32_t>((size_t)R * L + 1);  // task_pos
  c.take<int32_t>((size_t)R * L + 1);  // tok_pos
  return c.bytes();
}

omnimoe_status ep_pack(int dtype, int64_t L, int d, int hk, int R, int64_t n_per, const void* x, const int32_t* idx,
                       const float* gate, void* x_send, int32_t* rec_send, int32_t* inv, int32_t* offsets,
                       int64_t* counts, void* ws, cudaStream_t st) {
  Carver c(ws);
  int32_t* cnt = c.take<int32_t>((size_t)R * L);
  int32_t* has = c.take<int32_t>((size_t)R * L);
  int32_t* task_pos = c.take<int32_t>((size_t)R * L + 1);
  int32_t* tok_pos = c.take<int32_t>((size_t)R * L + 1);
  ep_count_kernel<<<grid_of(L, 128), 128, 0, st>>>(idx, L, hk, R, n_per, cnt, has);
  OMNI_CHECK_LAUNCH("ep_count_kernel");
  ep_scan_kernel<<<1, 1024, 0, st>>>(cnt, (int64_t)R * L, task_pos);
  OMNI_CHECK_LAUNCH("ep_scan_kernel(tasks)");
  ep_scan_kernel<<<1, 1024, 0, st>>>(has, (int64_t)R * L, tok_pos);
  OMNI_CHECK_LAUNCH("ep_scan_kernel(tokens)");
  if (dtype == OMNIMOE_BF16)
    ep_pack_kernel<__nv_bfloat16><<<grid_of(L * 32, 256), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), idx, gate, L, d, hk, R, n_per, task_pos, tok_pos,
        static_cast<__nv_bfloat16*>(x_send), rec_send, inv);
  else
    ep_pack_kernel<float><<<grid_of(L * 32, 256), 256, 0, st>>>(static_cast<const float*>(x), idx, gate, L, d, hk,
                                                                R, n_per, task_pos, tok_pos,
                                                                static_cast<float*>(x_send), rec_send, inv);
  OMNI_CHECK_LAUNCH("ep_pack_kernel");
  // offsets[0..R]: first send row (token) per destination; offsets[R+1..2R+1]: first record
  ep_offsets_kernel<<<1, 32, 0, st>>>(tok_pos, task_pos, L, R, offsets, counts);
  OMNI_CHECK_LAUNCH("ep_offsets_kernel");
  return OMNIMOE_OK;
}

omnimoe_status ep_unpack(const int32_t* rec, int64_t M, int R, const int64_t* task_off, const int64_t* tok_off,
                         int32_t* ids, float* gate, int32_t* tok, cudaStream_t st) {
  if (M == 0) return OMNIMOE_OK;
  ep_unpack_kernel<<<grid_of(M, 256), 256, 0, st>>>(rec, M, R, task_off, tok_off, ids, gate, tok);
  OMNI_CHECK_LAUNCH("ep_unpack_kernel");
  return OMNIMOE_OK;
}

omnimoe_status ep_combine(const void* y_ret, int bf16, const int32_t* inv, const int64_t* tok_off, int64_t L, int d,
                          int R, float* y, cudaStream_t st) {
  if (L == 0) return OMNIMOE_OK;
  if (bf16) ep_combine_kernel<true><<<grid_of(L * d / 4, 256), 256, 0, st>>>(y_ret, inv, tok_off, L, d, R, y);
  else ep_combine_kernel<false><<<grid_of(L * d / 4, 256), 256, 0, st>>>(y_ret, inv, tok_off, L, d, R, y);
  OMNI_CHECK_LAUNCH("ep_combine_kernel");
  return OMNIMOE_OK;
}

omnimoe_status ep_partials_bf16(const float* y, int64_t n, void* out, cudaStream_t st) {
  if (n == 0) return OMNIMOE_OK;
  ep_partials_kernel<<<grid_of(n / 4, 256), 256, 0, st>>>(reinterpret_cast<const float4*>(y), n / 4,
                                                          static_cast<uint2*>(out));
  OMNI_CHECK_LAUNCH("ep_partials_kernel");
  return OMNIMOE_OK;
}

}  // namespace omni
