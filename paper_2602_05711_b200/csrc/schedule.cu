// Expert-Centric Scheduling, steps a4-a5 of DESIGN.md.
//
// Tasks t = ((l*h)+head)*K + k arrive in token-major order (Eq.Tasks,
// PAPER:261-265).  a4: per-local-expert histogram, exclusive scan ->
// expert_offsets, compaction of active experts (E_active).
// a5, B = 1 (the expert-major plan): a counting sort -- each task claims a slot of its
// expert's segment [offsets[e], offsets[e+1]) with an atomic countdown (arbitrary order
// inside the segment), then every segment is sorted by task index, which restores the
// order a stable sort of the token-major task list gives (tokens ascending inside each
// expert segment, Eq.Sort with group size B = 1, reading Q14), and the plan arrays are
// written from it.  One pass over the tasks instead of the three (histogram + scatter)
// rounds of an 8-bit LSD radix sort.
// a5, B > 1: stable LSD radix sort (8-bit digits, "radix sort") of the (token
// block, group) keys with the task index as payload; stability over the token-major
// input gives tokens ascending inside each group.  Tasks outside the local expert range
// get the sentinel key and sort behind every segment.
// Everything is deterministic (no order-dependent atomics reach the output).
#include "schedule.cuh"

namespace omni {
namespace {

constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;
constexpr int kRadixThreads = 256, kRadixRounds = 16, kRadixTile = kRadixThreads * kRadixRounds;

// V order (SLICED executor): one warp per token stably partitions the token's
// tasks by band b = e / band_size (b = nb outside the local range); dest[t] = the
// task's V-order position, task_pair[dest].x = its local expert id (-1 outside),
// seg[l*(nb+1) + b] = start of segment (l, b).
__global__ void band_partition_kernel(const int32_t* __restrict__ ids, int64_t begin, int64_t n_loc,
                                      const int32_t* __restrict__ tok_off, int64_t hk, int64_t M, int64_t n_tok,
                                      int nb, int64_t band_size,
                                      int32_t* __restrict__ dest, int32_t* __restrict__ task_pair,
                                      int32_t* __restrict__ seg) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  // tok_off == nullptr: the default token of task t is t / hk
  auto toff = [&](int64_t l) { return tok_off ? (int64_t)tok_off[l] : std::min<int64_t>(l * hk, M); };
  if (gw == 0 && lane == 0) seg[n_tok * (nb + 1)] = (int32_t)toff(n_tok);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t l = gw; l < n_tok; l += nw) {
    const int beg = (int)toff(l), end = (int)toff(l + 1);
    auto band_of = [&](int t) {
      const int64_t e = (int64_t)ids[t] - begin;
      return (e >= 0 && e < n_loc) ? (int)(e / band_size) : nb;
    };
    int cnt = 0;  // lane b < nb+1 counts band b
    for (int t0 = beg; t0 < end; t0 += 32) {
      const int b = t0 + lane < end ? band_of(t0 + lane) : nb + 1;
      for (int q = 0; q <= nb; ++q) {
        const int c = __popc(__ballot_sync(0xffffffffu, b == q));
        if (lane == q) cnt += c;
      }
    }
    int incl = cnt;  // exclusive prefix over lanes 0..nb
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = beg + incl - cnt;  // lane q: next position of band q
    if (lane <= nb) seg[l * (nb + 1) + lane] = pos;
    for (int t0 = beg; t0 < end; t0 += 32) {
      const int t = t0 + lane;
      const int b = t < end ? band_of(t) : nb + 1;
      int q_pos = 0;
      for (int q = 0; q <= nb; ++q) {
        const unsigned m = __ballot_sync(0xffffffffu, b == q);
        const int base = __shfl_sync(0xffffffffu, pos, q);
        if (b == q) q_pos = base + __popc(m & lt);
        if (lane == q) pos += __popc(m);
      }
      if (t < end) {
        dest[t] = q_pos;
        task_pair[2 * (size_t)q_pos] = b < nb ? (int32_t)(ids[t] - begin) : -1;
      }
    }
  }
}

__global__ void hist_keys_kernel(const int32_t* __restrict__ ids, int64_t M, int64_t begin,
                                 int64_t n_loc, uint32_t* __restrict__ keys,
                                 int32_t* __restrict__ cnt, int32_t* __restrict__ task_pair) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = (int64_t)ids[t] - begin;
    const bool in = e >= 0 && e < n_loc;
    if (keys) keys[t] = in ? (uint32_t)e : (uint32_t)n_loc;
    if (task_pair) task_pair[2 * t] = in ? (int32_t)e : -1;  // one band: V order = task order
    if (in) atomicAdd(&cnt[e], 1);
  }
}

// off[l * stride] = first task of token l (tasks sorted by token), for l in
// [0, n_tokens]; thread t fills the offsets of the tokens in (token(t-1), token(t)].
// stride 2 (one band): off[2l + 1] = off[2(l+1)] too, i.e. segment (l, 0) is the
// whole token and segment (l, 1) (outside the range) is empty.
__global__ void token_offsets_kernel(int64_t M, const int32_t* __restrict__ token, int64_t hk, int64_t n_tokens,
                                     int32_t* __restrict__ off, int stride) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= M;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cur = t < M ? (token ? (int64_t)token[t] : t / hk) : n_tokens;
    const int64_t prev = t > 0 ? (token ? (int64_t)token[t - 1] : (t - 1) / hk) : -1;
    for (int64_t l = prev + 1; l <= cur && l <= n_tokens; ++l) {
      off[l * stride] = (int32_t)t;
      if (stride == 2 && l > 0) off[2 * l - 1] = (int32_t)t;
    }
  }
}

// block-wide exclusive scan of one value per thread; returns prefix, *total = sum
__device__ int block_exclusive_scan(int v, int* total, int* warp_sums) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) warp_sums[w] = x;
  __syncthreads();
  int wp = 0, tot = 0;
  for (int i = 0; i < nw; ++i) {
    if (i < w) wp += warp_sums[i];
    tot += warp_sums[i];
  }
  *total = tot;
  return wp + x - v;
}

// MODE 0: plain exclusive scan of in (out[i] = prefix);  MODE 1: compaction of
// nonzero entries (out[prefix] = i);  MODE 2: exclusive scan of (in > 0)
// written densely (out[i] = number of nonzero entries before i).
template <int MODE>
__global__ void __launch_bounds__(kScanThreads)
    scan_reduce_kernel(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ tile_sums) {
  __shared__ int ws[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int s = 0;
  for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
    const int64_t g = base + i;
    if (g < n) s += MODE ? (in[g] > 0) : in[g];
  }
  int tot;
  block_exclusive_scan(s, &tot, ws);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024)
    scan_tiles_kernel(int32_t* __restrict__ tile_sums, int nt, int32_t* __restrict__ total_out) {
  __shared__ int ws[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b = 0; b < nt; b += 1024) {
    const int i = b + threadIdx.x;
    const int v = i < nt ? tile_sums[i] : 0;
    int tot;
    const int ex = block_exclusive_scan(v, &tot, ws);
    if (i < nt) tile_sums[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

template <int MODE>
__global__ void __launch_bounds__(kScanThreads)
    scan_down_kernel(const int32_t* __restrict__ in, int64_t n, const int32_t* __restrict__ tile_off,
                     int32_t* __restrict__ out) {
  __shared__ int tile[kScanTile];
  __shared__ int ws[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
    const int64_t g = base + i;
    tile[i] = g < n ? (MODE ? (in[g] > 0) : in[g]) : 0;
  }
  __syncthreads();
  int v[kScanItems], s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = tile[threadIdx.x * kScanItems + j];
    s += v[j];
  }
  int tot;
  int run = block_exclusive_scan(s, &tot, ws) + tile_off[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t g = base + threadIdx.x * kScanItems + j;
    if (MODE != 1) {
      tile[threadIdx.x * kScanItems + j] = run;
    } else if (v[j] && g < n) {
      out[run] = (int32_t)g;
    }
    run += v[j];
  }
  if (MODE != 1) {
    __syncthreads();
    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads) {
      const int64_t g = base + i;
      if (g < n) out[g] = tile[i];
    }
  }
}

template <int MODE>
omnimoe_status scan(const int32_t* in, int64_t n, int32_t* out, int32_t* total, int32_t* tile_sums,
                    cudaStream_t st) {
  const int nt = (int)((n + kScanTile - 1) / kScanTile);
  if (nt == 0) return OMNIMOE_OK;
  scan_reduce_kernel<MODE><<<nt, kScanThreads, 0, st>>>(in, n, tile_sums);
  OMNI_CHECK_LAUNCH("scan_reduce_kernel");
  scan_tiles_kernel<<<1, 1024, 0, st>>>(tile_sums, nt, total);
  OMNI_CHECK_LAUNCH("scan_tiles_kernel");
  scan_down_kernel<MODE><<<nt, kScanThreads, 0, st>>>(in, n, tile_sums, out);
  OMNI_CHECK_LAUNCH("scan_down_kernel");
  return OMNIMOE_OK;
}

// ---- radix sort ------------------------------------------------------------
__global__ void __launch_bounds__(kRadixThreads)
    radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift, int nb,
                      int32_t* __restrict__ hist) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRadixTile;
  for (int i = threadIdx.x; i < kRadixTile; i += kRadixThreads) {
    const int64_t g = base + i;
    if (g < n) atomicAdd(&h[(keys[g] >> shift) & 255], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: a tile is consumed in rounds of 256 consecutive keys; inside a
// round, a key's destination = digit base + keys of the same digit in lower
// warps + same-digit lanes below it in its warp (__match_any_sync).
__global__ void __launch_bounds__(kRadixThreads)
    radix_scatter_kernel(const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
                         uint32_t* __restrict__ kout, int32_t* __restrict__ vout, int64_t n,
                         int shift, int nb, const int32_t* __restrict__ digit_off) {
  __shared__ int wcnt[kRadixThreads / 32][256];
  __shared__ int base[256];
  __shared__ int rtot[256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  base[tid] = digit_off[(int64_t)tid * nb + blockIdx.x];
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kRadixRounds; ++r) {
#pragma unroll
    for (int w = 0; w < kRadixThreads / 32; ++w) wcnt[w][tid] = 0;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * kRadixTile + (int64_t)r * kRadixThreads + tid;
    const bool valid = i < n;
    uint32_t key = 0;
    int32_t val = 0;
    int dig = 0, rank = 0;
    const unsigned mask = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      key = kin[i];
      val = vin ? vin[i] : (int32_t)i;
      dig = (key >> shift) & 255;
      const unsigned peers = __match_any_sync(mask, dig);
      rank = __popc(peers & lt);
      if (rank == 0) wcnt[warp][dig] = __popc(peers);
    }
    __syncthreads();
    {
      int s = 0;
#pragma unroll
      for (int w = 0; w < kRadixThreads / 32; ++w) {
        const int c = wcnt[w][tid];
        wcnt[w][tid] = s;
        s += c;
      }
      rtot[tid] = s;
    }
    __syncthreads();
    if (valid) {
      const int dest = base[dig] + wcnt[warp][dig] + rank;
      kout[dest] = key;
      vout[dest] = val;
    }
    __syncthreads();
    base[tid] += rtot[tid];
  }
}

// B > 1: replace each in-range key (local expert id) by its group
// q = rank_active(e) / B; out-of-range tasks keep a sentinel that
// sorts behind every group.
// With T_b token blocks the key is (block of t) * n_groups_max + q, so the sort
// is Eq.Sort applied to each block of tpb consecutive tasks in turn.
__global__ void group_keys_kernel(uint32_t* __restrict__ keys, int64_t M, int64_t n_loc,
                                  const int32_t* __restrict__ rank, int64_t B, int64_t tpb,
                                  uint32_t n_groups_max, uint32_t sentinel) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = keys[t];
    keys[t] = e < (uint32_t)n_loc ? (uint32_t)(t / tpb) * n_groups_max + (uint32_t)(rank[e] / B) : sentinel;
  }
}

// run boundaries of the sorted plan: position p starts a run if its group or
// its token differs from position p-1's.
__global__ void run_flags_kernel(const uint32_t* __restrict__ skeys, const int32_t* __restrict__ stok,
                                 int64_t M, const int32_t* __restrict__ m_loc_ptr,
                                 int32_t* __restrict__ flags) {
  const int64_t m_loc = *m_loc_ptr;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
       p += (int64_t)gridDim.x * blockDim.x)
    flags[p] = p < m_loc && (p == 0 || skeys[p] != skeys[p - 1] || stok[p] != stok[p - 1]);
}

__global__ void gather_plan_kernel(const int32_t* __restrict__ order, int64_t M,
                                   const int32_t* __restrict__ m_loc_ptr,
                                   const int32_t* __restrict__ token, const float* __restrict__ gate,
                                   const int32_t* __restrict__ ids, int64_t begin, int64_t hk,
                                   int32_t* __restrict__ sorted_token, float* __restrict__ sorted_gate,
                                   int32_t* __restrict__ sorted_expert, int32_t* __restrict__ sorted_task,
                                   const int32_t* __restrict__ dest, const uint32_t* __restrict__ skeys) {
  const int64_t m_loc = *m_loc_ptr;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m_loc;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = order[p];
    sorted_token[p] = token ? token[t] : (int32_t)(t / hk);
    sorted_gate[p] = gate[t];
    // B = 1: the sorted keys are the local expert ids (coalesced, instead of a gather)
    sorted_expert[p] = skeys ? (int32_t)skeys[p] : (int32_t)(ids[t] - begin);
    if (sorted_task) sorted_task[p] = dest ? dest[t] : t;
  }
}

// B = 1: task t -> a slot of its expert's segment (the countdown of cnt[e] gives slots
// n_e - 1 .. 0 in arbitrary order; segment_sort_kernel restores task order)
__global__ void count_scatter_kernel(const int32_t* __restrict__ ids, const float* __restrict__ gate, int64_t M,
                                     int64_t begin, int64_t n_loc, const int32_t* __restrict__ off,
                                     int32_t* __restrict__ cnt, int2* __restrict__ perm) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = (int64_t)ids[t] - begin;
    if (e >= 0 && e < n_loc) perm[off[e] + atomicSub(&cnt[e], 1) - 1] = make_int2((int32_t)t, __float_as_int(gate[t]));
  }
}

// a segment of n <= 16 (task, gate) pairs sorted by task index in registers: 16-input
// bitonic network on 64-bit words (task index in the high half: the indices are distinct)
__device__ __forceinline__ void cswap64(unsigned long long& x, unsigned long long& y, bool up) {
  const bool sw = up ? (x > y) : (x < y);
  const unsigned long long tx = x;
  x = sw ? y : x;
  y = sw ? tx : y;
}
__device__ __forceinline__ void sort16(unsigned long long (&v)[16]) {
#pragma unroll
  for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int l = i ^ j;
        if (l > i) cswap64(v[i], v[l], (i & k) == 0);
      }
}
__device__ __forceinline__ unsigned long long pack_tg(int2 p) {
  return ((unsigned long long)(uint32_t)p.x << 32) | (uint32_t)p.y;
}

// one warp per 32 consecutive active experts.  Their segments are contiguous in the plan
// ([off[e_0], off[e_31 + 1]): inactive experts have empty segments), so the warp stages
// the region's (task, gate) pairs in shared memory with coalesced loads, every lane sorts
// its expert's segment (n <= 16, E n = eta ~ 8) in registers, and the warp writes the
// region's plan entries with coalesced stores.  Regions over the staging capacity and
// segments over 16 tasks take the per-lane / queued paths.
constexpr int kSegCap = 512;  // pairs staged per warp (E region = 32 eta ~ 256)
__global__ void __launch_bounds__(256)
    segment_sort_kernel(const int32_t* __restrict__ active, const int32_t* __restrict__ n_active_p,
                        const int32_t* __restrict__ off, const int2* __restrict__ perm,
                        const int32_t* __restrict__ token, int64_t hk, const int32_t* __restrict__ dest,
                        int32_t* __restrict__ sorted_token, float* __restrict__ sorted_gate,
                        int32_t* __restrict__ sorted_expert, int32_t* __restrict__ sorted_task,
                        int32_t* __restrict__ big_list, int32_t* __restrict__ big_count) {
  __shared__ int2 stage[8][kSegCap];
  __shared__ int32_t eid[8][kSegCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int2* st = stage[wib];
  int32_t* ei = eid[wib];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int na = *n_active_p;
  for (int i = lane; i < kSegCap; i += 32) ei[i] = -1;
  __syncwarp();
  auto emit = [&](int64_t p, int2 tg, int e) {
    const int32_t t = tg.x;
    sorted_token[p] = token ? token[t] : (int32_t)(t / hk);
    sorted_gate[p] = __int_as_float(tg.y);
    sorted_expert[p] = e;
    if (sorted_task) sorted_task[p] = dest ? dest[t] : t;
  };
  for (int64_t base = gw * 32; base < na; base += nw * 32) {
    const bool valid = base + lane < na;
    const int e = valid ? active[base + lane] : 0;
    const int a = valid ? off[e] : 0, n = valid ? off[e + 1] - a : 0;
    const int A0 = __shfl_sync(0xffffffffu, a, 0);
    const int last = (int)(na - 1 - base < 31 ? na - 1 - base : 31);
    const int A1 = __shfl_sync(0xffffffffu, a + n, last);
    const bool big = n > 16;
    if (big) big_list[atomicAdd(big_count, 1)] = e;
    if (A1 - A0 <= kSegCap) {
      for (int p = A0 + lane; p < A1; p += 32) st[p - A0] = perm[p];
      __syncwarp();
      if (!big && n > 0) {
        unsigned long long v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = i < n ? pack_tg(st[a - A0 + i]) : ~0ull;
        sort16(v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i < n) {
            st[a - A0 + i] = make_int2((int32_t)(v[i] >> 32), (int32_t)(uint32_t)v[i]);
            ei[a - A0 + i] = e;
          }
      }
      __syncwarp();
      for (int p = A0 + lane; p < A1; p += 32) {
        // big segments are written by segment_sort_big_kernel
        if (ei[p - A0] >= 0) emit(p, st[p - A0], ei[p - A0]);
      }
      __syncwarp();
      for (int p = A0 + lane; p < A1; p += 32) ei[p - A0] = -1;  // reset for the next region
      __syncwarp();
    } else if (!big && n > 0) {  // region over capacity: this lane's segment from global memory
      unsigned long long v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = i < n ? pack_tg(perm[a + i]) : ~0ull;
      sort16(v);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < n) emit(a + i, make_int2((int32_t)(v[i] >> 32), (int32_t)(uint32_t)v[i]), e);
    }
  }
}

// segments longer than 16 tasks (the tail of the per-expert load: ~0.4 % of the active
// experts at eta = 8; or skewed routing): one WARP per segment; the rank of every task
// index is the number of smaller ones, counted with shuffles over 32-wide chunks of the
// segment -- O(n^2 / 32) per segment, which the load statistics keep small
__global__ void __launch_bounds__(256)
    segment_sort_big_kernel(const int32_t* __restrict__ big_list, const int32_t* __restrict__ big_count,
                            const int32_t* __restrict__ off, const int2* __restrict__ perm,
                            const int32_t* __restrict__ token, int64_t hk, const int32_t* __restrict__ dest,
                            int32_t* __restrict__ sorted_token, float* __restrict__ sorted_gate,
                            int32_t* __restrict__ sorted_expert, int32_t* __restrict__ sorted_task) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int nbig = *big_count;
  for (int64_t q = gw; q < nbig; q += nw) {
    const int e = big_list[q];
    const int a = off[e], n = off[e + 1] - a;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int i = c0 + lane;
      const int2 tg = i < n ? perm[a + i] : make_int2(INT32_MAX, 0);
      int rank = 0;
      for (int j0 = 0; j0 < n; j0 += 32) {
        const int32_t u = j0 + lane < n ? perm[a + j0 + lane].x : INT32_MAX;
#pragma unroll
        for (int k = 0; k < 32; ++k) rank += __shfl_sync(0xffffffffu, u, k) < tg.x;
      }
      if (i < n) {
        const int64_t p = a + rank;
        sorted_token[p] = token ? token[tg.x] : (int32_t)(tg.x / hk);
        sorted_gate[p] = __int_as_float(tg.y);
        sorted_expert[p] = e;
        if (sorted_task) sorted_task[p] = dest ? dest[tg.x] : tg.x;
      }
    }
  }
}

// load metrics of a plan: per block, in a fixed order, the number of
// used experts and sum_{c>0} (c/M) log(n_loc c / M) over the block's experts
__global__ void __launch_bounds__(256)
    load_stats_kernel(const int32_t* __restrict__ off, int64_t n_loc, double* __restrict__ partial) {
  __shared__ double su[256], sk[256];
  const double M = (double)off[n_loc];
  double used = 0.0, kl = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_loc; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = off[e + 1] - off[e];
    if (c > 0) {
      const double z = (double)c / M;
      used += 1.0;
      kl += z * log((double)n_loc * z);
    }
  }
  su[threadIdx.x] = used;
  sk[threadIdx.x] = kl;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      su[threadIdx.x] += su[threadIdx.x + o];
      sk[threadIdx.x] += sk[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = su[0];
    partial[2 * blockIdx.x + 1] = sk[0];
  }
}

__global__ void load_stats_final_kernel(const double* __restrict__ partial, int nblk, int64_t n_loc,
                                        const int32_t* __restrict__ off, double* __restrict__ out) {
  double u = 0.0, k = 0.0;
  for (int b = 0; b < nblk; ++b) {
    u += partial[2 * b];
    k += partial[2 * b + 1];
  }
  const bool any = off[n_loc] > 0;
  out[0] = any ? u / (double)n_loc : 0.0;
  out[1] = any ? k : 0.0;
}

int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::min<int64_t>(std::max<int64_t>(b, 1), num_sms() * 16);
}

}  // namespace

size_t load_stats_ws_bytes() { return 2 * num_sms() * 2 * sizeof(double); }

omnimoe_status load_stats_run(const omnimoe_plan& plan, double* out, void* ws, cudaStream_t st) {
  const int64_t n_loc = plan.expert_end - plan.expert_begin;
  const int nblk = num_sms() * 2;
  load_stats_kernel<<<nblk, 256, 0, st>>>(plan.expert_offsets, n_loc, static_cast<double*>(ws));
  OMNI_CHECK_LAUNCH("load_stats_kernel");
  load_stats_final_kernel<<<1, 1, 0, st>>>(static_cast<const double*>(ws), nblk, n_loc, plan.expert_offsets, out);
  OMNI_CHECK_LAUNCH("load_stats_final_kernel");
  return OMNIMOE_OK;
}

size_t schedule_ws_bytes(int64_t M, int64_t n_loc) {
  Carver c(nullptr);
  const int64_t nb = (M + kRadixTile - 1) / kRadixTile;
  c.take<int32_t>(n_loc + 1);                                 // cnt
  c.take<int32_t>(n_loc + 1);                                 // rank among active
  c.take<uint32_t>(M); c.take<uint32_t>(M);                   // keys ping/pong
  c.take<int32_t>(M); c.take<int32_t>(M);                     // vals ping/pong
  c.take<int32_t>(256 * nb);                                  // radix hist
  const int64_t scan_n = std::max<int64_t>(std::max<int64_t>(n_loc + 1, 256 * nb), M);
  c.take<int32_t>((scan_n + kScanTile - 1) / kScanTile + 1);  // tile sums
  c.take<int32_t>(M + 2);                                     // per-token task offsets (V order)
  c.take<int32_t>(std::max<int64_t>(M, 1));                   // V-order destination of each task
  return c.bytes();
}

omnimoe_status schedule_run(int64_t M, const int32_t* ids, const float* gate, const int32_t* token,
                            int64_t hk, const omnimoe_plan& plan, int64_t B, int64_t Tb, int64_t n_bands,
                            void* ws, cudaStream_t st) {
  const int64_t n_loc = plan.expert_end - plan.expert_begin;
  const int64_t nb = (M + kRadixTile - 1) / kRadixTile;
  if (B > 1 && M > 0) {  // (token block, group) keys are uint32 with n_keys as the out-of-range sentinel
    const int64_t L = (M + hk - 1) / hk;
    const int64_t tb = std::max<int64_t>(1, std::min<int64_t>(Tb, L));
    const int64_t ngm = (n_loc + B - 1) / B;
    if (tb * ngm >= (int64_t(1) << 32) - 1) {
      set_error("schedule: token_blocks (" + std::to_string(tb) + ") x groups (" + std::to_string(ngm) +
                ") must be < 2^32 - 1");
      return OMNIMOE_ERR_SHAPE;
    }
  }
  Carver c(ws);
  int32_t* cnt = c.take<int32_t>(n_loc + 1);
  int32_t* rank = c.take<int32_t>(n_loc + 1);
  uint32_t* k0 = c.take<uint32_t>(M);
  uint32_t* k1 = c.take<uint32_t>(M);
  int32_t* v0 = c.take<int32_t>(M);
  int32_t* v1 = c.take<int32_t>(M);
  int32_t* hist = c.take<int32_t>(256 * nb);
  const int64_t scan_n = std::max<int64_t>(std::max<int64_t>(n_loc + 1, 256 * nb), M);
  int32_t* tiles = c.take<int32_t>((scan_n + kScanTile - 1) / kScanTile + 1);
  int32_t* tok_off = c.take<int32_t>(M + 2);
  int32_t* dest = c.take<int32_t>(std::max<int64_t>(M, 1));
  const bool vorder = plan.task_pair && plan.token_offsets && plan.sorted_task;

  if (cudaMemsetAsync(cnt, 0, (n_loc + 1) * sizeof(int32_t), st) != cudaSuccess ||
      (B > 1 && cudaMemsetAsync(plan.n_runs, 0, sizeof(int32_t), st) != cudaSuccess)) {
    set_error("schedule: memset failed");
    return OMNIMOE_ERR_CUDA;
  }
  if (M > 0) {
    hist_keys_kernel<<<grid_for(M, 256), 256, 0, st>>>(ids, M, plan.expert_begin, n_loc, B > 1 ? k0 : nullptr, cnt,
                                                       vorder && n_bands == 1 ? plan.task_pair : nullptr);
    OMNI_CHECK_LAUNCH("hist_keys_kernel");
  }
  if (vorder) {  // the SLICED executor's (token, band) order
    const int64_t n_tok = plan.n_tokens > 0 ? plan.n_tokens : (M + hk - 1) / hk;
    if (n_tok > M + 1) {
      set_error("schedule: n_tokens larger than the task count + 1 is not supported");
      return OMNIMOE_ERR_SHAPE;
    }
    if (n_bands == 1) {  // V order = task order; out-of-range tasks carry expert -1
      token_offsets_kernel<<<grid_for(M + 1, 256), 256, 0, st>>>(M, token, hk, n_tok, plan.token_offsets, 2);
      OMNI_CHECK_LAUNCH("token_offsets_kernel");
    } else {
      if (token) {
        token_offsets_kernel<<<grid_for(M + 1, 256), 256, 0, st>>>(M, token, hk, n_tok, tok_off, 1);
        OMNI_CHECK_LAUNCH("token_offsets_kernel");
      }
      const int64_t band_size = (n_loc + n_bands - 1) / n_bands;
      band_partition_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((n_tok + 7) / 8, num_sms() * 16)), 256, 0,
                              st>>>(ids, plan.expert_begin, n_loc, token ? tok_off : nullptr, hk, M, n_tok,
                                    (int)n_bands, band_size, dest, plan.task_pair, plan.token_offsets);
      OMNI_CHECK_LAUNCH("band_partition_kernel");
    }
  }
  // a4: offsets (exclusive scan of counts; entry n_loc holds the total m_loc)
  OMNI_TRY(scan<0>(cnt, n_loc + 1, plan.expert_offsets, nullptr, tiles, st));
  // a4: active-expert compaction and |E_active|
  OMNI_TRY(scan<1>(cnt, n_loc, plan.active, plan.n_active, tiles, st));
  if (M == 0) return OMNIMOE_OK;
  if (B == 1) {  // a5 as a counting sort + per-segment sort (see the top of this file)
    int2* perm = reinterpret_cast<int2*>(k0);  // k0 and k1 are adjacent: M (task, gate) pairs
    int32_t* big = v0;                 // queued long segments (<= n_active entries <= M)
    int32_t* big_count = cnt + n_loc;  // cnt[n_loc] is 0 after the scans and free now
    count_scatter_kernel<<<grid_for(M, 256), 256, 0, st>>>(ids, gate, M, plan.expert_begin, n_loc,
                                                          plan.expert_offsets, cnt, perm);
    OMNI_CHECK_LAUNCH("count_scatter_kernel");
    const int32_t* dst = vorder && n_bands > 1 ? dest : nullptr;
    int32_t* stask = vorder ? plan.sorted_task : nullptr;
    segment_sort_kernel<<<num_sms() * 4, 256, 0, st>>>(plan.active, plan.n_active, plan.expert_offsets, perm, token, hk,
                                                  dst, plan.sorted_token, plan.sorted_gate, plan.sorted_expert, stask,
                                                  big, big_count);
    OMNI_CHECK_LAUNCH("segment_sort_kernel");
    segment_sort_big_kernel<<<num_sms() * 4, 256, 0, st>>>(big, big_count, plan.expert_offsets, perm, token, hk, dst,
                                                 plan.sorted_token, plan.sorted_gate, plan.sorted_expert, stask);
    OMNI_CHECK_LAUNCH("segment_sort_big_kernel");
    return OMNIMOE_OK;
  }
  // a4: group of each expert = rank among the active experts / B
  int64_t n_keys = n_loc;  // largest key value (the sentinel)
  if (B > 1) {
    OMNI_TRY(scan<2>(cnt, n_loc, rank, nullptr, tiles, st));
    const int64_t ngm = (n_loc + B - 1) / B;
    const int64_t L = (M + hk - 1) / hk;
    Tb = std::max<int64_t>(1, std::min<int64_t>(Tb, L));
    const int64_t tpb = hk * ((L + Tb - 1) / Tb);  // tasks per block, whole tokens
    n_keys = Tb * ngm;
    group_keys_kernel<<<grid_for(M, 256), 256, 0, st>>>(k0, M, n_loc, rank, B, tpb, (uint32_t)ngm,
                                                        (uint32_t)n_keys);
    OMNI_CHECK_LAUNCH("group_keys_kernel");
  }
  // a5: stable LSD radix sort of the keys (sentinel included), task index payload
  int bits = 1;
  while ((int64_t(1) << bits) <= n_keys) ++bits;
  const int passes = (bits + 7) / 8;
  uint32_t *kin = k0, *kout = k1;
  int32_t *vin = nullptr, *vout = v0;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = 8 * ps;
    radix_hist_kernel<<<(int)nb, kRadixThreads, 0, st>>>(kin, M, shift, (int)nb, hist);
    OMNI_CHECK_LAUNCH("radix_hist_kernel");
    OMNI_TRY(scan<0>(hist, 256 * nb, hist, nullptr, tiles, st));
    radix_scatter_kernel<<<(int)nb, kRadixThreads, 0, st>>>(kin, vin, kout, vout, M, shift, (int)nb, hist);
    OMNI_CHECK_LAUNCH("radix_scatter_kernel");
    std::swap(kin, kout);
    vin = vout;
    vout = (vout == v0) ? v1 : v0;
  }
  const int32_t* m_loc = plan.expert_offsets + n_loc;
  gather_plan_kernel<<<grid_for(M, 256), 256, 0, st>>>(vin, M, m_loc, token, gate, ids, plan.expert_begin, hk,
                                                      plan.sorted_token, plan.sorted_gate, plan.sorted_expert,
                                                      vorder ? plan.sorted_task : nullptr, vorder && n_bands > 1 ? dest : nullptr,
                                                      B > 1 ? nullptr : kin);
  OMNI_CHECK_LAUNCH("gather_plan_kernel");
  if (B > 1) {
    // runs: (group, token) boundaries of the sorted plan, compacted to run_offsets
    int32_t* flags = reinterpret_cast<int32_t*>(kout);  // free buffer (kin holds the sorted keys)
    run_flags_kernel<<<grid_for(M, 256), 256, 0, st>>>(kin, plan.sorted_token, M, m_loc, flags);
    OMNI_CHECK_LAUNCH("run_flags_kernel");
    OMNI_TRY(scan<1>(flags, M, plan.run_offsets, plan.n_runs, tiles, st));
  }
  return OMNIMOE_OK;
}

}  // namespace omni
