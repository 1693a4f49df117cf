// Cartesian Product Router selection, steps a2 + a3 of DESIGN.md.
//
// One CTA per token-head (persistent grid).  Input: the exact logits of the
// token-head, s_r[0..N_r) then s_c[0..N_c) (a1, reading Q9).
//
//  a2  per half: keys ord32(s) << 32 | ~index (one integer compare = value desc,
//      index asc); radix-select the k'-th largest (k' = min(K+1, n)), compact the
//      k' survivors in index order, bitonic-sort them; logsumexp of the half
//      (Eq.LSM) for the reported scores.
//  a3  candidates = cells whose 1-based half ranks satisfy a*b <= K+1 (every
//      cell of the exact top K+1 is one); exact key of a cell =
//      TwoSum(s_r[i], s_c[j]) as a 128-bit integer (ord64(hi), ord32(lo) << 32 |
//      ~flat id) so that one compare = (exact key desc, flat id asc) (Q7);
//      radix-select the (K+1)-th largest, compact, bitonic-sort the K+1;
//      gates = softmax over the first K exact keys (Eq.Gate);
//      score = key - lse_r - lse_c (Eq.S, Q8).
// All reductions use fixed trees, compaction follows index order: the output is
// bitwise deterministic and independent of L and of the batch.
#include "router.cuh"

namespace omni {
namespace {

constexpr int kSelThreads = 256;
constexpr int kWarps = kSelThreads / 32;

struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ bool gt(const U128& x, const U128& y) {
  return x.hi > y.hi || (x.hi == y.hi && x.lo > y.lo);
}
__device__ __forceinline__ bool gt(uint64_t x, uint64_t y) { return x > y; }
__device__ __forceinline__ uint32_t byte_of(uint64_t k, int pos) { return (uint32_t)(k >> (8 * pos)) & 255u; }
__device__ __forceinline__ uint32_t byte_of(const U128& k, int pos) {
  return pos >= 8 ? (uint32_t)(k.hi >> (8 * (pos - 8))) & 255u : (uint32_t)(k.lo >> (8 * pos)) & 255u;
}
// key restricted to the bytes above `pos` equals the prefix?
__device__ __forceinline__ bool prefix_eq(uint64_t k, uint64_t pre, int pos) {
  return pos >= 7 ? true : (k >> (8 * (pos + 1))) == (pre >> (8 * (pos + 1)));
}
__device__ __forceinline__ bool prefix_eq(const U128& k, const U128& pre, int pos) {
  if (pos >= 15) return true;
  if (pos >= 8) return (k.hi >> (8 * (pos - 7))) == (pre.hi >> (8 * (pos - 7)));
  return k.hi == pre.hi && (pos >= 7 || (k.lo >> (8 * (pos + 1))) == (pre.lo >> (8 * (pos + 1))));
}
__device__ __forceinline__ void set_byte(uint64_t& k, int pos, uint32_t b) { k |= (uint64_t)b << (8 * pos); }
__device__ __forceinline__ void set_byte(U128& k, int pos, uint32_t b) {
  if (pos >= 8) k.hi |= (uint64_t)b << (8 * (pos - 8));
  else k.lo |= (uint64_t)b << (8 * pos);
}
__device__ __forceinline__ bool ge(const U128& x, const U128& y) { return !gt(y, x); }
__device__ __forceinline__ bool ge(uint64_t x, uint64_t y) { return x >= y; }

struct SelShared {
  int hist[256];
  int red_i[kWarps];
  float red_f[kWarps];
  int bcast[4];
};

// MSB-first radix select of the `want`-th largest of n unique keys produced by
// keyf(i).  Returns a threshold thr such that exactly `want` keys satisfy
// key >= thr.  Requires 1 <= want <= n.
template <class KeyT, int NBYTES, class KeyF>
__device__ KeyT radix_select(int n, int want, KeyF keyf, SelShared& sh) {
  KeyT pre{};
  int remaining = want;
  const int lane = threadIdx.x & 31;
  for (int pos = NBYTES - 1; pos >= 0; --pos) {
    for (int i = threadIdx.x; i < 256; i += kSelThreads) sh.hist[i] = 0;
    __syncthreads();
    const int nloop = (n + kSelThreads - 1) / kSelThreads * kSelThreads;
    for (int i = threadIdx.x; i < nloop; i += kSelThreads) {
      uint32_t dig = 256;
      if (i < n) {
        const KeyT k = keyf(i);
        if (prefix_eq(k, pre, pos)) dig = byte_of(k, pos);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, dig);
      if (dig < 256 && lane == __ffs(peers) - 1) atomicAdd(&sh.hist[dig], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // suffix sums over bins 255..0; lane j owns bins [255-8j-7, 255-8j]
      int c[8], s = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        c[t] = sh.hist[255 - 8 * lane - t];
        s += c[t];
      }
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int above = incl - s;  // keys in bins higher than this lane's bins
      int found = -1, fabove = 0, fcnt = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (found < 0 && above < remaining && above + c[t] >= remaining) {
          found = 255 - 8 * lane - t;
          fabove = above;
          fcnt = c[t];
        }
        above += c[t];
      }
      const unsigned who = __ballot_sync(0xffffffffu, found >= 0);
      const int src = __ffs(who) - 1;
      found = __shfl_sync(0xffffffffu, found, src);
      fabove = __shfl_sync(0xffffffffu, fabove, src);
      fcnt = __shfl_sync(0xffffffffu, fcnt, src);
      if (lane == 0) {
        sh.bcast[0] = found;
        sh.bcast[1] = fabove;
        sh.bcast[2] = fcnt;
      }
    }
    __syncthreads();
    const int b = sh.bcast[0];
    remaining -= sh.bcast[1];
    set_byte(pre, pos, (uint32_t)b);
    const bool done = sh.bcast[2] == remaining;  // the whole bucket is selected
    __syncthreads();
    if (done) break;  // lower bytes of pre stay 0: key >= pre selects the bucket
  }
  return pre;
}

// deterministic compaction of the keys >= thr (index order) into out[0..)
template <class KeyT, class KeyF>
__device__ void compact_ge(int n, KeyT thr, KeyF keyf, KeyT* out, SelShared& sh) {
  const int per = (n + kSelThreads - 1) / kSelThreads;
  const int b0 = threadIdx.x * per, b1 = min(n, b0 + per);
  int cnt = 0;
  for (int i = b0; i < b1; ++i) cnt += ge(keyf(i), thr);
  // block exclusive scan of cnt
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh.red_i[w] = x;
  __syncthreads();
  int off = 0;
  for (int i = 0; i < w; ++i) off += sh.red_i[i];
  off += x - cnt;
  for (int i = b0; i < b1; ++i) {
    const KeyT k = keyf(i);
    if (ge(k, thr)) out[off++] = k;
  }
  __syncthreads();
}

template <class K>
__device__ void bitonic_desc(K* a, int n) {  // n a power of two; padding must hold minimal keys
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += kSelThreads) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const K p = a[lo], q = a[hi];
        if (desc ? gt(q, p) : gt(p, q)) {
          a[lo] = q;
          a[hi] = p;
        }
      }
      __syncthreads();
    }
}

__device__ float block_sum(float v, SelShared& sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh.red_f[w] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < kWarps; ++i) r += sh.red_f[i];
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint64_t half_key(float v, uint32_t i) {
  v = v + 0.0f;  // -0.0 -> +0.0: equal values compare equal
  return ((uint64_t)ord32(v) << 32) | (uint64_t)(0xFFFFFFFFu - i);
}
__device__ __forceinline__ float half_val(uint64_t k) { return ord32_inv((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t half_idx(uint64_t k) { return 0xFFFFFFFFu - (uint32_t)k; }
__device__ __forceinline__ double ord64_inv(uint64_t u) {
  return __longlong_as_double((long long)((u & 0x8000000000000000ull) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u));
}

// exact key of cell (i, j) from its two logits (TwoSum; lo is exact in fp32)
__device__ __forceinline__ U128 cell_key(float vr, float vc, uint32_t n) {
  const double a = (double)vr, b = (double)vc;
  double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  s = s + 0.0;
  const float ef = (float)e + 0.0f;
  return U128{ord64(s), ((uint64_t)ord32(ef) << 32) | (uint64_t)(0xFFFFFFFFu - n)};
}
__device__ __forceinline__ double key_value(const U128& k) {  // hi + lo as a double (gates only)
  return ord64_inv(k.hi) + (double)ord32_inv((uint32_t)(k.lo >> 32));
}

// sorts the top k1 keys of one half into out[0..k1) (padded to pk1 with zeros)
__device__ void half_topk(const float* lg, int n, int k1, int pk1, uint64_t* raw, uint64_t* out,
                          SelShared& sh, float* lse) {
  for (int i = threadIdx.x; i < n; i += kSelThreads) raw[i] = half_key(lg[i], (uint32_t)i);
  __syncthreads();
  auto keyf = [raw](int i) { return raw[i]; };
  uint64_t thr = 0;
  if (k1 < n) thr = radix_select<uint64_t, 8>(n, k1, keyf, sh);
  compact_ge(n, thr, keyf, out, sh);
  for (int i = k1 + threadIdx.x; i < pk1; i += kSelThreads) out[i] = 0ull;
  __syncthreads();
  bitonic_desc(out, pk1);
  const float mx = half_val(out[0]);
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += kSelThreads) s += __expf(lg[i] - mx);
  s = block_sum(s, sh);
  *lse = mx + __logf(s);
}

__global__ void __launch_bounds__(kSelThreads)
    select_kernel(SelectParams p, const float* __restrict__ logits, int32_t* __restrict__ idx,
                  float* __restrict__ gate, float* __restrict__ score) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ SelShared sh;
  // layout: sel (U128[pkeep]) | raw (u64[max(nr, nc)]) | kr (u64[pkr]) | kc (u64[pkc]) | cand (u32[C])
  U128* sel = reinterpret_cast<U128*>(smem);
  uint64_t* raw = reinterpret_cast<uint64_t*>(sel + p.pkeep);
  uint64_t* kr = raw + max(p.n_rows, p.n_cols);
  uint64_t* kc = kr + p.pkr;
  uint32_t* cand = reinterpret_cast<uint32_t*>(kc + p.pkc);

  const int R = p.n_rows + p.n_cols;
  const int K1 = p.top_k + 1;
  // candidate (a, b) pairs, the same for every token-head: row ranks a admit
  // b < min(kc1, K1 / (a + 1)) (0-based ranks); packed a << 16 | b
  if (threadIdx.x == 0) sh.bcast[3] = 0;
  __syncthreads();
  for (int a = threadIdx.x; a < p.kr1; a += kSelThreads) {
    int off = 0;
    for (int t = 0; t < a; ++t) off += min(p.kc1, K1 / (t + 1));
    const int nb = min(p.kc1, K1 / (a + 1));
    for (int b = 0; b < nb; ++b) cand[off + b] = ((uint32_t)a << 16) | (uint32_t)b;
  }
  __syncthreads();
  const int C = p.C;
  const int keep = min(K1, C);

  for (int th = blockIdx.x; th < p.T; th += gridDim.x) {
    const float* lg = logits + (size_t)th * R;
    float lse_r, lse_c;
    half_topk(lg, p.n_rows, p.kr1, p.pkr, raw, kr, sh, &lse_r);
    half_topk(lg + p.n_rows, p.n_cols, p.kc1, p.pkc, raw, kc, sh, &lse_c);
    const uint32_t Nc = (uint32_t)p.n_cols;
    auto ckey = [kr, kc, cand, Nc](int c) {
      const uint32_t ab = cand[c];
      const uint64_t ka = kr[ab >> 16], kb = kc[ab & 0xFFFF];
      return cell_key(half_val(ka), half_val(kb), half_idx(ka) * Nc + half_idx(kb));
    };
    U128 thr{0ull, 0ull};
    if (keep < C) thr = radix_select<U128, 16>(C, keep, ckey, sh);
    compact_ge(C, thr, ckey, sel, sh);
    for (int i = keep + threadIdx.x; i < p.pkeep; i += kSelThreads) sel[i] = U128{0ull, 0ull};
    __syncthreads();
    bitonic_desc(sel, p.pkeep);
    // ---- gates: softmax over the K selected exact keys (Eq.Gate) ----
    const double k1v = key_value(sel[0]);
    float es = 0.f;
    for (int k = threadIdx.x; k < p.top_k; k += kSelThreads) es += expf((float)(key_value(sel[k]) - k1v));
    es = block_sum(es, sh);
    const float inv = 1.0f / es;
    for (int k = threadIdx.x; k < p.top_k; k += kSelThreads) {
      const U128 q = sel[k];
      const double kv = key_value(q);
      const size_t o = (size_t)th * p.top_k + k;
      idx[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)q.lo);
      gate[o] = expf((float)(kv - k1v)) * inv;
      if (score) score[o] = (float)(kv - (double)lse_r - (double)lse_c);
    }
    __syncthreads();
  }
}

int pow2ceil(int v) {
  int q = 1;
  while (q < v) q <<= 1;
  return q;
}

}  // namespace

// host --------------------------------------------------------------------
omnimoe_status select_params(const omnimoe_dims& d, int64_t T, SelectParams* p, size_t* smem) {
  p->T = (int)T;
  p->n_rows = (int)d.n_rows;
  p->n_cols = (int)d.n_cols;
  p->top_k = (int)d.top_k;
  const int64_t K1 = d.top_k + 1;
  p->kr1 = (int)std::min<int64_t>(K1, d.n_rows);
  p->kc1 = (int)std::min<int64_t>(K1, d.n_cols);
  int64_t C = 0;
  for (int64_t a = 1; a <= p->kr1; ++a) C += std::min<int64_t>(p->kc1, K1 / a);
  p->C = (int)C;
  p->pkr = pow2ceil(p->kr1);
  p->pkc = pow2ceil(p->kc1);
  p->pkeep = pow2ceil((int)std::min<int64_t>(K1, C));
  if (d.n_rows > 65535 || d.n_cols > 65535) {
    set_error("route: grid halves must be <= 65535");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  *smem = (size_t)p->pkeep * 16 + (size_t)std::max(p->n_rows, p->n_cols) * 8 +
          (size_t)(p->pkr + p->pkc) * 8 + (size_t)C * 4 + 16;
  if (*smem > 225 * 1024) {
    set_error("route: selection working set (" + std::to_string(*smem) +
              " bytes: K+1 sorted keys, both halves, " + std::to_string(C) +
              " product candidates) exceeds shared memory");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  return OMNIMOE_OK;
}

omnimoe_status launch_select(const SelectParams& p, size_t smem, const float* logits, int32_t* idx,
                             float* gate, float* score, cudaStream_t st) {
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    if (cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
      set_error("route: cannot set select_kernel shared memory");
      return OMNIMOE_ERR_CUDA;
    }
    attr = smem;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel, kSelThreads, smem);
  const int grid = std::min(p.T, kSMs * std::max(per_sm, 1));
  if (grid <= 0) return OMNIMOE_OK;
  select_kernel<<<grid, kSelThreads, smem, st>>>(p, logits, idx, gate, score);
  OMNI_CHECK_LAUNCH("select_kernel");
  return OMNIMOE_OK;
}

}  // namespace omni
