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
#include <cstdlib>

#include "router.cuh"

namespace omni {
namespace {

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

// ---------------------------------------------------------------------------
// Cooperative primitives of a selection group: G = 32 (one warp per token-head,
// __syncwarp only) or G = 256 (one CTA per token-head).  Each group owns a
// SelShared and its key buffers in shared memory.
template <int G>
struct Grp {
  static constexpr int kW = G / 32;
  __device__ static __forceinline__ int tid() { return G == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x; }
  __device__ static __forceinline__ void sync() {
    if (G == 32) __syncwarp();
    else __syncthreads();
  }
};

template <int G>
struct SelShared {
  int hist[256];
  int red_i[G / 32];
  float red_f[G / 32];
  int bcast[4];
  U128 red_k[G / 32];
  U128 kmin;
};

__device__ __forceinline__ U128 shfl_xor_key(const U128& k, int o) {
  return U128{__shfl_xor_sync(0xffffffffu, k.hi, o), __shfl_xor_sync(0xffffffffu, k.lo, o)};
}
__device__ __forceinline__ uint64_t shfl_xor_key(uint64_t k, int o) { return __shfl_xor_sync(0xffffffffu, k, o); }
__device__ __forceinline__ U128 to128(const U128& k) { return k; }
__device__ __forceinline__ U128 to128(uint64_t k) { return U128{0ull, k}; }
__device__ __forceinline__ void from128(const U128& s, U128& k) { k = s; }
__device__ __forceinline__ void from128(const U128& s, uint64_t& k) { k = s.lo; }

// smallest of a[0..n) (keys unique), moved to a[n-1]; returns it
template <int G, class KeyT>
__device__ KeyT extract_min_last(KeyT* a, int n, SelShared<G>& sh) {
  using g = Grp<G>;
  KeyT m;
  from128(U128{~0ull, ~0ull}, m);  // threads without elements offer the largest key
  for (int i = g::tid(); i < n; i += G)
    if (gt(m, a[i])) m = a[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const KeyT q = shfl_xor_key(m, o);
    if (gt(m, q)) m = q;
  }
  if (G > 32) {
    if ((threadIdx.x & 31) == 0) sh.red_k[threadIdx.x >> 5] = to128(m);
    g::sync();
    from128(sh.red_k[0], m);
    for (int i = 1; i < g::kW; ++i) {
      KeyT q;
      from128(sh.red_k[i], q);
      if (gt(m, q)) m = q;
    }
  }
  for (int i = g::tid(); i < n - 1; i += G) {  // exactly one element equals m
    const KeyT v = a[i];
    if (!gt(v, m) && !gt(m, v)) {
      a[i] = a[n - 1];
      a[n - 1] = v;
    }
  }
  g::sync();
  return m;
}

// MSB-first radix select of the `want`-th largest of n unique keys produced by
// keyf(i).  Returns a threshold thr such that exactly `want` keys satisfy
// key >= thr.  Requires 1 <= want <= n.
template <int G, class KeyT, int NBYTES, class KeyF>
__device__ KeyT radix_select(int n, int want, KeyF keyf, SelShared<G>& sh) {
  using g = Grp<G>;
  KeyT pre{};
  int remaining = want;
  const int lane = threadIdx.x & 31;
  for (int pos = NBYTES - 1; pos >= 0; --pos) {
    for (int i = g::tid(); i < 256; i += G) sh.hist[i] = 0;
    g::sync();
    const int nloop = (n + G - 1) / G * G;
    for (int i = g::tid(); i < nloop; i += G) {
      uint32_t dig = 256;
      if (i < n) {
        const KeyT k = keyf(i);
        if (prefix_eq(k, pre, pos)) dig = byte_of(k, pos);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, dig);
      if (dig < 256 && lane == __ffs(peers) - 1) atomicAdd(&sh.hist[dig], __popc(peers));
    }
    g::sync();
    if (g::tid() < 32) {
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
      int above = incl - s;
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
    g::sync();
    const int b = sh.bcast[0];
    remaining -= sh.bcast[1];
    set_byte(pre, pos, (uint32_t)b);
    const bool done = sh.bcast[2] == remaining;  // the whole bucket is selected
    g::sync();
    if (done) break;  // lower bytes of pre stay 0: key >= pre selects the bucket
  }
  return pre;
}

// deterministic compaction of the keys >= thr (STRICT: > thr) in index order into out[0..)
template <int G, bool STRICT, class KeyT, class KeyF>
__device__ void compact_ge(int n, KeyT thr, KeyF keyf, KeyT* out, SelShared<G>& sh) {
  using g = Grp<G>;
  const int per = (n + G - 1) / G;
  const int b0 = g::tid() * per, b1 = min(n, b0 + per);
  auto take = [&](const KeyT& k) { return STRICT ? gt(k, thr) : ge(k, thr); };
  int cnt = 0;
  for (int i = b0; i < b1; ++i) cnt += take(keyf(i));
  const int lane = threadIdx.x & 31;
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  int off = x - cnt;
  if (G > 32) {
    const int w = threadIdx.x >> 5;
    if (lane == 31) sh.red_i[w] = x;
    g::sync();
    for (int i = 0; i < w; ++i) off += sh.red_i[i];
  }
  for (int i = b0; i < b1; ++i) {
    const KeyT k = keyf(i);
    if (take(k)) out[off++] = k;
  }
  g::sync();
}

// Pair i of a stage compares a[lo], a[lo + stride], lo = 2i - (i mod stride).  For
// stride <= 32 the pairs of the 32 consecutive i of one warp stay inside one 64-key
// block, so consecutive warp-local stages only need __syncwarp; a block barrier is
// needed only around stages with stride >= 64.
template <int G, class K>
__device__ void bitonic_desc(K* a, int n) {  // n a power of two; padding must hold minimal keys
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = Grp<G>::tid(); i < (n >> 1); i += G) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const K p = a[lo], q = a[hi];
        if (desc ? gt(q, p) : gt(p, q)) {
          a[lo] = q;
          a[hi] = p;
        }
      }
      const int next = stride > 1 ? stride >> 1 : size;  // stride of the next stage
      if (G > 32 && (stride >= 64 || next >= 64 || (stride == 1 && size == n))) __syncthreads();
      else __syncwarp();
    }
}

// pow2 size used to sort the top `keep` of n unique keys: with a radix-selected
// threshold the keep-th key is extracted and placed last, the keep-1 larger are sorted
__host__ __device__ inline int sort_len(int keep, int n) {
  int want = keep < n ? keep - 1 : keep, q = 1;
  while (q < want) q <<= 1;
  return q;
}

// top `keep` of n keys produced by keyf, sorted descending into out[0..keep)
// (out holds max(sort_len, keep) entries; entries beyond keep are scratch)
template <int G, class KeyT, int NBYTES, class KeyF>
__device__ void top_sorted(int n, int keep, KeyF keyf, KeyT* out, SelShared<G>& sh) {
  const int len = sort_len(keep, n);
  if (keep < n) {
    const KeyT thr = radix_select<G, KeyT, NBYTES>(n, keep, keyf, sh);
    compact_ge<G, false>(n, thr, keyf, out, sh);             // exactly the top `keep` keys
    const KeyT last = extract_min_last<G>(out, keep, sh);    // the keep-th key, not sorted
    for (int i = keep - 1 + Grp<G>::tid(); i < len; i += G) out[i] = KeyT{};
    Grp<G>::sync();
    bitonic_desc<G>(out, len);
    if (Grp<G>::tid() == 0) out[keep - 1] = last;
  } else {
    compact_ge<G, false>(n, KeyT{}, keyf, out, sh);          // all keys (every key is > 0)
    for (int i = keep + Grp<G>::tid(); i < len; i += G) out[i] = KeyT{};
    Grp<G>::sync();
    bitonic_desc<G>(out, len);
  }
  Grp<G>::sync();
}

template <int G>
__device__ float group_sum(float v, SelShared<G>& sh) {
  v = warp_sum(v);
  if (G == 32) return v;
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh.red_f[w] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < G / 32; ++i) r += sh.red_f[i];
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

// the top k1 keys of one half, sorted, into out[0..k1); *lse = logsumexp of the half
template <int G>
__device__ void half_topk(const float* __restrict__ lg, int n, int k1, uint64_t* out, SelShared<G>& sh,
                          float* lse) {
  auto keyf = [lg](int i) { return half_key(lg[i], (uint32_t)i); };
  top_sorted<G, uint64_t, 8>(n, k1, keyf, out, sh);
  const float mx = half_val(out[0]);
  float s = 0.f;
  for (int i = Grp<G>::tid(); i < n; i += G) s += __expf(lg[i] - mx);
  s = group_sum<G>(s, sh);
  *lse = mx + __logf(s);
}

// ---------------------------------------------------------------------------
// Small K (K + 1 <= 32): one WARP per token-head, no block barriers.  The t-th
// largest key of a list is found by t rounds of "largest key below the previous
// one" (each lane scans its strided share, then a shuffle max); lane t keeps it.
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ U128 warp_max_u128(U128 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const U128 q = shfl_xor_key(v, o);
    if (gt(q, v)) v = q;
  }
  return v;
}

// lane t (< k1) returns the t-th largest half key of lg[0..n); *lse = logsumexp
__device__ uint64_t warp_half_topk(const float* __restrict__ lg, int n, int k1, float* lse) {
  const int lane = threadIdx.x & 31;
  uint64_t mine = 0, prev = ~0ull;
  for (int t = 0; t < k1; ++t) {
    uint64_t best = 0;
    for (int i = lane; i < n; i += 32) {
      const uint64_t k = half_key(lg[i], (uint32_t)i);
      if (k < prev && k > best) best = k;
    }
    best = warp_max_u64(best);
    if (lane == t) mine = best;
    prev = best;
  }
  const float mx = half_val(__shfl_sync(0xffffffffu, mine, 0));
  float s = 0.f;
  for (int i = lane; i < n; i += 32) s += __expf(lg[i] - mx);
  s = warp_sum(s);
  *lse = mx + __logf(s);
  return mine;
}

// per-group shared memory: SelShared | kr (pkr u64) | kc (pkc u64) | sel (pkeep U128)
template <int G>
__host__ __device__ inline size_t group_bytes(const SelectParams& p) {
  size_t b = (sizeof(SelShared<G>) + 15) / 16 * 16;
  b += (size_t)(p.pkr + p.pkc) * 8;
  b = (b + 15) / 16 * 16;
  return b + (size_t)p.pkeep * 16;
}

template <int G>
__global__ void __launch_bounds__(G > 256 ? G : 256)
    select_kernel(SelectParams p, const float* __restrict__ logits, int32_t* __restrict__ idx,
                  float* __restrict__ gate, float* __restrict__ score) {
  extern __shared__ __align__(16) uint8_t smem[];
  // CTA-wide candidate table (a, b) with a*b <= K+1 (0-based ranks), the same for every token-head
  uint32_t* cand = reinterpret_cast<uint32_t*>(smem);
  const size_t cand_bytes = ((size_t)p.C * 4 + 15) / 16 * 16;
  const int K1 = p.top_k + 1;
  // row a holds min(kc1, K1 / (a+1)) candidates; its offset is a prefix sum computed by
  // thread 0 into the table's tail (scratch, overwritten below in index order)
  int* row_off = reinterpret_cast<int*>(smem + ((size_t)p.C * 4 + 15) / 16 * 16) ;
  if (threadIdx.x == 0) {
    int off = 0;
    for (int a = 0; a < p.kr1; ++a) {
      row_off[a] = off;
      off += min(p.kc1, K1 / (a + 1));
    }
  }
  __syncthreads();
  for (int a = threadIdx.x; a < p.kr1; a += blockDim.x) {
    const int off = row_off[a], nb = min(p.kc1, K1 / (a + 1));
    for (int b = 0; b < nb; ++b) cand[off + b] = ((uint32_t)a << 16) | (uint32_t)b;
  }
  __syncthreads();
  const int gid = threadIdx.x / G, ngroups = blockDim.x / G;
  uint8_t* base = smem + cand_bytes + (size_t)gid * group_bytes<G>(p);
  SelShared<G>& sh = *reinterpret_cast<SelShared<G>*>(base);
  uint64_t* kr = reinterpret_cast<uint64_t*>(base + (sizeof(SelShared<G>) + 15) / 16 * 16);
  uint64_t* kc = kr + p.pkr;
  U128* sel = reinterpret_cast<U128*>(base + ((sizeof(SelShared<G>) + 15) / 16 * 16 +
                                              (size_t)(p.pkr + p.pkc) * 8 + 15) / 16 * 16);
  const int R = p.n_rows + p.n_cols;
  const int C = p.C;
  const int keep = min(p.top_k, C);  // exact logits: no K+1-th key (gap) is needed
  const uint32_t Nc = (uint32_t)p.n_cols;
  for (int th = blockIdx.x * ngroups + gid; th < p.T; th += gridDim.x * ngroups) {
    const float* lg = logits + (size_t)th * R;
    float lse_r, lse_c;
    half_topk<G>(lg, p.n_rows, p.kr1, kr, sh, &lse_r);
    half_topk<G>(lg + p.n_rows, p.n_cols, p.kc1, kc, sh, &lse_c);
    auto ckey = [kr, kc, cand, Nc](int c) {
      const uint32_t ab = cand[c];
      const uint64_t ka = kr[ab >> 16], kb = kc[ab & 0xFFFF];
      return cell_key(half_val(ka), half_val(kb), half_idx(ka) * Nc + half_idx(kb));
    };
    if (p.sorted) {
      top_sorted<G, U128, 16>(C, keep, ckey, sel, sh);
    } else {  // the K largest, in candidate order (no sort; cell (0,0) is the maximum)
      const U128 thr = keep < C ? radix_select<G, U128, 16>(C, keep, ckey, sh) : U128{0ull, 0ull};
      compact_ge<G, false>(C, thr, ckey, sel, sh);
    }
    // ---- gates: softmax over the K selected exact keys (Eq.Gate) ----
    const double k1v = key_value(p.sorted ? sel[0] : ckey(0));
    float es = 0.f;
    for (int k = Grp<G>::tid(); k < p.top_k; k += G) es += expf((float)(key_value(sel[k]) - k1v));
    es = group_sum<G>(es, sh);
    const float inv = 1.0f / es;
    for (int k = Grp<G>::tid(); k < p.top_k; k += G) {
      const U128 q = sel[k];
      const double kv = key_value(q);
      const size_t o = (size_t)th * p.top_k + k;
      idx[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)q.lo);
      gate[o] = expf((float)(kv - k1v)) * inv;
      if (score) score[o] = (float)(kv - (double)lse_r - (double)lse_c);
    }
    Grp<G>::sync();
  }
}

// ---------------------------------------------------------------------------
// Large K, candidate-order output (the layer path, sorted == 0): one WARP per
// token-head, no block barriers.  Selections use bucket refinement on 64-bit
// order-preserving integer keys: each pass histograms the keys inside the current
// range [lo, hi] into 256 buckets of width 2^shift (span >> shift < 256), keeps the
// bucket holding the want-th largest, and stops when the whole range is taken or
// holds one key value (ties, resolved on the full key) -- at most 8 passes.
struct WPred {  // selected <=> bk > thr || (bk == thr && full >= kmin)
  uint64_t thr;
  U128 kmin;
};
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// items: slots m = 0..nslot-1 of this lane; bkf(m, ok) -> bucket key (ok = item
// exists); fullf(m) -> full key (needed only for ties).  lo0: a lower bound of the
// want-th largest bucket key (items below it are never selected).
// loop over this lane's item slots: fully unrolled over MAXS register slots, or a
// plain loop over nslot (MAXS = 0)
#define OMNI_SLOT_LOOP(m)                                                          \
  _Pragma("unroll") for (int m##_o = 0; m##_o < (MAXS ? MAXS : 1); ++m##_o)        \
    for (int m = (MAXS ? m##_o : 0); m < (MAXS ? m##_o + 1 : nslot); ++m)          \
      if (MAXS && m >= nslot) {                                                    \
      } else
template <int MAXS = 0, class BkF, class FullF>
__device__ WPred warp_select_top(int nslot, BkF bkf, FullF fullf, int want, uint64_t lo0, int* hist) {
  const int lane = threadIdx.x & 31;
  uint64_t lo = ~0ull, hi = 0;
  int cnt = 0;
  OMNI_SLOT_LOOP(m) {
    bool ok;
    const uint64_t k = bkf(m, ok);
    if (ok && k >= lo0) {
      lo = min(lo, k);
      hi = max(hi, k);
      ++cnt;
    }
  }
  lo = warp_min_u64(lo);
  hi = warp_max_u64(hi);
  cnt = warp_sum(cnt);
  int r = want;
  while (r < cnt && lo < hi) {
    const uint64_t span = hi - lo;
    const int shift = max(0, 64 - __clzll((long long)span) - 8);  // span >> shift < 256
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0;
    __syncwarp();
    OMNI_SLOT_LOOP(m) {
      bool ok;
      const uint64_t k = bkf(m, ok);
      if (ok && k >= lo && k <= hi) atomicAdd(&hist[(int)((k - lo) >> shift)], 1);
    }
    __syncwarp();
    // suffix counts from the top bucket: lane j owns buckets 255-8j .. 255-8j-7
    int c[8], sum = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      c[t] = hist[255 - 8 * lane - t];
      sum += c[t];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int above = incl - sum, found = -1, fabove = 0, fcnt = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (found < 0 && above < r && above + c[t] >= r) {
        found = 255 - 8 * lane - t;
        fabove = above;
        fcnt = c[t];
      }
      above += c[t];
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, found >= 0)) - 1;
    const int b = __shfl_sync(0xffffffffu, found, src);
    r -= __shfl_sync(0xffffffffu, fabove, src);
    cnt = __shfl_sync(0xffffffffu, fcnt, src);
    const uint64_t nlo = lo + ((uint64_t)b << shift);
    const uint64_t w = (shift == 0) ? 0ull : ((1ull << shift) - 1ull);
    hi = (hi - nlo > w) ? nlo + w : hi;
    lo = nlo;
    __syncwarp();  // the histogram is cleared again by the next pass
  }
  WPred p;
  p.thr = lo;
  p.kmin = U128{0ull, 0ull};
  if (r < cnt) {  // one bucket-key value, more items than wanted: the r largest full keys
    U128 prev{~0ull, ~0ull};
    for (int t = 0; t < r; ++t) {
      U128 best{0ull, 0ull};
      OMNI_SLOT_LOOP(m) {
        bool ok;
        const uint64_t k = bkf(m, ok);
        if (ok && k == lo) {
          const U128 f = fullf(m);
          if (gt(prev, f) && gt(f, best)) best = f;
        }
      }
      prev = warp_max_u128(best);
    }
    p.kmin = prev;
  }
  return p;
}

// bitonic sort (descending) of a[0..n), n a power of two, by one warp
__device__ void warp_bitonic_desc(uint64_t* a, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const uint64_t p = a[lo], q = a[hi];
        if (desc ? q > p : p > q) {
          a[lo] = q;
          a[hi] = p;
        }
      }
      __syncwarp();
    }
}

// descending sort of n <= kBucketSortMax unique half keys a[0..n) by one warp: a
// 256-bucket counting sort on the key's value (bucket = floor((v - vmin) * 256 /
// (vmax - vmin)), monotone in the key), then each key's rank inside its bucket by
// comparison with the bucket's other keys.  Work ~ sum over buckets of size^2, so it
// declines (returns false, a[] untouched) when that exceeds the bitonic network's cost.
// cur, st: 256 ints each (the per-warp histogram and the refinement list's space).
constexpr int kBucketSortMax = 512;
__device__ bool warp_bucket_sort_desc(uint64_t* a, int n, int* cur, int* st) {
  constexpr int J = kBucketSortMax / 32;
  const int lane = threadIdx.x & 31;
  uint64_t kk[J];
  float vmax = -INFINITY, vmin = INFINITY;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int i = lane + 32 * j;
    kk[j] = i < n ? a[i] : 0ull;
    if (i < n) {
      const float v = half_val(kk[j]);
      vmax = fmaxf(vmax, v);
      vmin = fminf(vmin, v);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
  }
  const float span = vmax - vmin;
  const float scale = (span > 0.f && span < INFINITY) ? 256.f / span : 0.f;
  // NaN (inf * 0) lands in bucket 0 through fmaxf; every step is monotone in v
  auto bucket = [&](uint64_t k) { return (int)fminf(255.f, fmaxf(0.f, (half_val(k) - vmin) * scale)); };
#pragma unroll
  for (int t = 0; t < 8; ++t) cur[lane * 8 + t] = 0;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < J; ++j)
    if (lane + 32 * j < n) atomicAdd(&cur[bucket(kk[j])], 1);
  __syncwarp();
  // descending: bucket 255 first; lane j owns buckets 255-8j .. 255-8j-7
  int c[8], sum = 0, sq = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    c[t] = cur[255 - 8 * lane - t];
    sum += c[t];
    sq += c[t] * c[t];
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  // the bitonic network costs ~log2(P)^2 / 2 compare-exchange steps of P / 64 per lane
  if (warp_sum(sq) > 24 * n) return false;
  int run = incl - sum;
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    st[255 - 8 * lane - t] = run;
    cur[255 - 8 * lane - t] = run;
    run += c[t];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < J; ++j)
    if (lane + 32 * j < n) a[atomicAdd(&cur[bucket(kk[j])], 1)] = kk[j];
  __syncwarp();
  int fp[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    fp[j] = -1;
    if (lane + 32 * j < n) {
      const int b = bucket(kk[j]), s0 = st[b], e0 = cur[b];
      int r = 0;
      for (int q = s0; q < e0; ++q) r += a[q] > kk[j];
      fp[j] = s0 + r;
    }
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < J; ++j)
    if (fp[j] >= 0) a[fp[j]] = kk[j];
  __syncwarp();
  return true;
}

// the top k1 half keys of lg[0..n), sorted descending into out[0..P)
// (P = pow2 >= k1, padded with 0 -- unless the bucket sort took them: then only
// out[0..k1) is written); returns logsumexp of the half if want_lse.  st: 256 ints
// for the bucket sort, or null (bitonic network only)
__device__ float warp_half_sorted(const float* __restrict__ lg, int n, int k1, int P, uint64_t* out, int* hist,
                                  bool want_lse, int* st = nullptr) {
  const int lane = threadIdx.x & 31;
  const int nslot = (n + 31) >> 5;
  auto bkf = [&](int m, bool& ok) {  // the half's logits stay in L1 over the passes
    const int i = lane + 32 * m;
    ok = i < n;
    return ok ? half_key(lg[i], (uint32_t)i) : 0ull;
  };
  WPred p;
  p.thr = 0;
  p.kmin = U128{0ull, 0ull};
  if (k1 < n)
    p = warp_select_top(nslot, bkf, [&](int m) { bool ok; return U128{bkf(m, ok), 0ull}; }, k1, 0ull, hist);
  // compact the selected keys (bucket keys are unique: bk >= thr) in slot order
  int base = 0;
  for (int m = 0; m < nslot; ++m) {
    bool ok;
    const uint64_t k = bkf(m, ok);
    const bool sel = ok && (k1 >= n || k >= p.thr);
    const unsigned bal = __ballot_sync(0xffffffffu, sel);
    if (sel) out[base + __popc(bal & ((1u << lane) - 1u))] = k;
    base += __popc(bal);
  }
  float lse = 0.f;
  if (want_lse) {  // before the sort, so that v[] is dead while the keys are in registers
    float mx = -INFINITY;
    for (int i = lane; i < n; i += 32) mx = fmaxf(mx, lg[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int i = lane; i < n; i += 32) sum += __expf(lg[i] - mx);
    lse = mx + __logf(warp_sum(sum));
  }
  __syncwarp();
  if (st && k1 <= kBucketSortMax && warp_bucket_sort_desc(out, k1, hist, st)) return lse;
  for (int i = k1 + lane; i < P; i += 32) out[i] = 0ull;
  __syncwarp();
  // bitonic network in shared memory (measured faster than a register-resident bitonic
  // sort, 1.24 vs 1.50 ms at C3a)
  warp_bitonic_desc(out, P);
  return lse;
}

// lane t (< k1 <= 32) returns the t-th largest half key of lg[0..n); *lse = logsumexp.
// Long halves (n > 256): bucket selection of the top k1 + a 32-key warp sort; short
// halves: k1 rounds of "largest key below the previous one".
__device__ uint64_t warp_half_topk_any(const float* __restrict__ lg, int n, int k1, float* lse, int* hist,
                                       uint64_t* srt) {
  if (n <= 256) return warp_half_topk(lg, n, k1, lse);
  const int lane = threadIdx.x & 31;
  warp_half_sorted(lg, n, k1, 32, srt, hist, false);
  const uint64_t mine = lane < k1 ? srt[lane] : 0ull;
  const float mx = half_val(__shfl_sync(0xffffffffu, srt[0], 0));
  __syncwarp();
  float sm = 0.f;
  for (int i = lane; i < n; i += 32) sm += __expf(lg[i] - mx);
  *lse = mx + __logf(warp_sum(sm));
  return mine;
}

// N4 fused path: lane t (< k1) returns the t-th largest key of the half's two epilogue
// lists (the top kp of each 48-column half of the GEMM's tiles, gemm_i8_topk_kernel); the
// half's logsumexp from their (max, sum exp) pairs
__device__ uint64_t warp_half_topk_fused(const uint64_t* __restrict__ c2, int kp, int k1,
                                         const float2* __restrict__ pp, float* lse) {
  const int lane = threadIdx.x & 31;
  const uint64_t a = lane < 2 * kp ? c2[lane] : 0ull;
  const uint64_t b = lane + 32 < 2 * kp ? c2[lane + 32] : 0ull;
  uint64_t prev = ~0ull, mine = 0ull;
  for (int t = 0; t < k1; ++t) {
    uint64_t best = a < prev ? a : 0ull;
    if (b < prev && b > best) best = b;
    best = warp_max_u64(best);
    if (lane == t) mine = best;
    prev = best;
  }
  if (pp) {
    const float2 p0 = pp[0], p1 = pp[1];
    const float M = fmaxf(p0.x, p1.x);
    const float sum = (p0.x == -INFINITY ? 0.f : p0.y * __expf(p0.x - M)) + (p1.x == -INFINITY ? 0.f : p1.y * __expf(p1.x - M));
    *lse = M + __logf(sum);
  }
  return mine;
}

__global__ void __launch_bounds__(256)
    select_warp_kernel(SelectParams p, const float* __restrict__ logits, int32_t* __restrict__ idx,
                       float* __restrict__ gate, float* __restrict__ score, const uint64_t* __restrict__ fcand,
                       const float2* __restrict__ fpart, int kp, int n_heads, const int32_t* __restrict__ fcounts,
                       const int32_t* __restrict__ fbad) {
  __shared__ uint32_t cand[1024];
  __shared__ int hist_all[8][256];      // per-warp bucket histograms (long halves)
  __shared__ uint64_t sorted_all[8][32];  // per-warp top-k1 keys of a half
  const int K1 = p.top_k + 1;
  if (threadIdx.x == 0) {
    int off = 0;
    for (int a = 0; a < p.kr1; ++a) {
      const int nb = min(p.kc1, K1 / (a + 1));
      for (int b = 0; b < nb; ++b) cand[off++] = ((uint32_t)a << 16) | (uint32_t)b;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * (int64_t)blockDim.x) >> 5);
  const int R = p.n_rows + p.n_cols;
  const int C = p.C, keep = min(K1, C);
  const uint32_t Nc = (uint32_t)p.n_cols;
  for (int th = gw; th < p.T; th += nw) {
    const float* lg = logits + (size_t)th * R;
    float lse_r = 0.f, lse_c = 0.f;
    int* hist = hist_all[(threadIdx.x >> 5) & 7];
    uint64_t* srt = sorted_all[(threadIdx.x >> 5) & 7];
    // the fused lists, unless a flag sent this token's logits (or every token's) through the
    // fp64 kernel
    bool fused = fcand != nullptr && fcounts[1] == 0;
    if (fused) {
      const int l = th / n_heads, nbad = fcounts[0];
      for (int j = 0; j < nbad; ++j) fused = fused && fbad[j] != l;
    }
    uint64_t kr, kc;
    if (fused) {
      const size_t base = (size_t)th * 2;  // (token, head) -> halves 2 * head, 2 * head + 1
      kr = warp_half_topk_fused(fcand + base * 2 * kp, kp, p.kr1, fpart ? fpart + base * 2 : nullptr, &lse_r);
      kc = warp_half_topk_fused(fcand + (base + 1) * 2 * kp, kp, p.kc1, fpart ? fpart + (base + 1) * 2 : nullptr,
                                &lse_c);
    } else {
      kr = warp_half_topk_any(lg, p.n_rows, p.kr1, &lse_r, hist, srt);
      kc = warp_half_topk_any(lg + p.n_rows, p.n_cols, p.kc1, &lse_c, hist, srt);
    }
    // candidate keys, at most ceil(C / 32) per lane (C <= 32 * (ln 32 + 1) < 160)
    U128 ck[5];
    const int per = (C + 31) / 32;
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      const int c = lane + 32 * m;
      const uint32_t ab = (m < per && c < C) ? cand[c] : 0u;
      const uint64_t ka = __shfl_sync(0xffffffffu, kr, (int)(ab >> 16));
      const uint64_t kb = __shfl_sync(0xffffffffu, kc, (int)(ab & 0xFFFF));
      ck[m] = (m < per && c < C) ? cell_key(half_val(ka), half_val(kb), half_idx(ka) * Nc + half_idx(kb))
                                 : U128{0ull, 0ull};
    }
    // the top `keep` candidates; lane t keeps the t-th
    U128 mine{0ull, 0ull}, prev{~0ull, ~0ull};
    for (int t = 0; t < keep; ++t) {
      U128 best{0ull, 0ull};
#pragma unroll
      for (int m = 0; m < 5; ++m)
        if (gt(prev, ck[m]) && gt(ck[m], best)) best = ck[m];
      best = warp_max_u128(best);
      if (lane == t) mine = best;
      prev = best;
    }
    // gates: softmax over the first K keys (Eq.Gate)
    const double k1v = key_value(U128{__shfl_sync(0xffffffffu, mine.hi, 0), __shfl_sync(0xffffffffu, mine.lo, 0)});
    const double kv = key_value(mine);
    const float ev = lane < p.top_k ? expf((float)(kv - k1v)) : 0.f;
    const float es = warp_sum(ev);
    if (lane < p.top_k) {
      const size_t o = (size_t)th * p.top_k + lane;
      idx[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)mine.lo);
      gate[o] = ev / es;
      if (score) score[o] = (float)(kv - (double)lse_r - (double)lse_c);
    }
  }
}

// smem: cand[C] (a << 16 | b, (a+1)(b+1) <= K) | per warp: kr[Pr], kc[Pc] (u64), hist[256],
// the refinement list (kListCap keys + candidate indices)
constexpr int kListCap = 256;
// the candidate table: rows a in order, columns b < min(kc, K / (a+1)); one 1024-thread
// block (kr <= 1024): row lengths, a block scan, then one warp per row writes its entries
__global__ void __launch_bounds__(1024) cand_table_kernel(int K, int kr, int kc, uint32_t* __restrict__ cand) {
  __shared__ int off[1025];
  __shared__ int wsum[32];
  const int a = threadIdx.x, lane = a & 31, w = a >> 5;
  const int nb = a < kr ? min(kc, K / (a + 1)) : 0;
  int inc = nb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  int base = 0;
  for (int i = 0; i < w; ++i) base += wsum[i];
  off[a] = base + inc - nb;
  __syncthreads();
  for (int r = w; r < kr; r += 32) {
    const int n = min(kc, K / (r + 1)), o = off[r];
    for (int b = lane; b < n; b += 32) cand[o + b] = ((uint32_t)r << 16) | (uint32_t)b;
  }
}

// CAND_SMEM: the candidate table is copied into shared memory (when it fits next to two
// CTAs' per-warp buffers); otherwise it is read from global memory through L1
template <bool CAND_SMEM>
__global__ void __launch_bounds__(256, 2)
    select_bucket_kernel(SelectParams p, int C, int Pr, int Pc, const uint32_t* __restrict__ cand_g,
                         const float* __restrict__ logits, int32_t* __restrict__ idx, float* __restrict__ gate,
                         float* __restrict__ score) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int K = p.top_k;
  const int kr = min(K, p.n_rows), kc = min(K, p.n_cols);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t cand_bytes = CAND_SMEM ? ((size_t)C * 4 + 15) / 16 * 16 : 0;
  const uint32_t* cand = cand_g;
  if (CAND_SMEM) {
    uint32_t* cs = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < C; i += blockDim.x) cs[i] = cand_g[i];
    __syncthreads();
    cand = cs;
  }
  const size_t per_warp = (size_t)(Pr + Pc) * 8 + 256 * 4 + kListCap * 12;
  uint8_t* base = smem + cand_bytes + (size_t)wid * per_warp;
  uint64_t* skr = reinterpret_cast<uint64_t*>(base);
  uint64_t* skc = skr + Pr;
  int* hist = reinterpret_cast<int*>(skc + Pc);
  const int R = p.n_rows + p.n_cols;
  const uint32_t Nc = (uint32_t)p.n_cols;
  const int nslot = (C + 31) >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wid, nw = gridDim.x * (blockDim.x >> 5);
  for (int th = gw; th < p.T; th += nw) {
    const float* lg = logits + (size_t)th * R;
    // the bucket sort's bucket starts go in the refinement list's space (hist + 256)
    const float lse_r = warp_half_sorted(lg, p.n_rows, kr, Pr, skr, hist, score != nullptr, hist + 256);
    const float lse_c = warp_half_sorted(lg + p.n_rows, p.n_cols, kc, Pc, skc, hist, score != nullptr, hist + 256);
    // sorted keys -> (value bits, index) pairs, read with one 8-byte load per half
    for (int a = lane; a < kr; a += 32) {
      const uint64_t k = skr[a];
      skr[a] = ((uint64_t)half_idx(k) << 32) | __float_as_uint(half_val(k));
    }
    for (int b = lane; b < kc; b += 32) {
      const uint64_t k = skc[b];
      skc[b] = ((uint64_t)half_idx(k) << 32) | __float_as_uint(half_val(k));
    }
    __syncwarp();
    auto hi_of = [&](int c, uint32_t& id, float& vr, float& vc) {
      const uint32_t ab = CAND_SMEM ? cand[c] : __ldg(cand + c);
      const uint2 ra = reinterpret_cast<const uint2*>(skr)[ab >> 16];
      const uint2 cb = reinterpret_cast<const uint2*>(skc)[ab & 0xFFFF];
      vr = __uint_as_float(ra.x);
      vc = __uint_as_float(cb.x);
      id = ra.y * Nc + cb.y;
      return ((double)vr + (double)vc) + 0.0;
    };
    auto bkf = [&](int m, bool& ok) {
      const int c = lane + 32 * m;
      ok = c < C;
      uint32_t id;
      float vr, vc;
      return ok ? ord64(hi_of(c, id, vr, vc)) : 0ull;
    };
    auto fullf = [&](int m) {
      uint32_t id;
      float vr, vc;
      hi_of(lane + 32 * m, id, vr, vc);
      return cell_key(vr, vc, id);
    };
    auto val_r = [&](int a) { return (double)__uint_as_float((uint32_t)skr[a]); };
    auto val_c = [&](int b) { return (double)__uint_as_float((uint32_t)skc[b]); };
    // lower bound of the K-th largest key: for A rows and B = ceil(K/A) columns, the
    // A*B >= K cells of the block all have keys >= s_r[A-1] + s_c[B-1]
    uint64_t lb = 0;
    for (int A = 1 + lane; A <= kr; A += 32) {
      const int B = (K + A - 1) / A;
      if (B <= kc) lb = max(lb, ord64((val_r(A - 1) + val_c(B - 1)) + 0.0));
    }
    lb = warp_max_u64(lb);
    const uint64_t kmax = ord64((val_r(0) + val_c(0)) + 0.0);  // cell (0, 0) holds the largest key
    // first bucket pass over [lb, kmax] on all candidates, then the bucket holding the
    // K-th key is compacted into a short list and refined there
    WPred sel;
    {
      const uint64_t span = kmax - lb;
      const int shift = span ? max(0, 64 - __clzll((long long)span) - 8) : 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0;
      __syncwarp();
      for (int m = 0; m < nslot; ++m) {
        bool ok;
        const uint64_t k = bkf(m, ok);
        if (ok && k >= lb) atomicAdd(&hist[(int)((k - lb) >> shift)], 1);
      }
      __syncwarp();
      int c8[8], sum = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        c8[t] = hist[255 - 8 * lane - t];
        sum += c8[t];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int above = incl - sum, found = -1, fabove = 0, fcnt = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (found < 0 && above < K && above + c8[t] >= K) {
          found = 255 - 8 * lane - t;
          fabove = above;
          fcnt = c8[t];
        }
        above += c8[t];
      }
      const int src = __ffs(__ballot_sync(0xffffffffu, found >= 0)) - 1;
      const int bstar = __shfl_sync(0xffffffffu, found, src);
      const int r = K - __shfl_sync(0xffffffffu, fabove, src);
      const int cnt = __shfl_sync(0xffffffffu, fcnt, src);
      const uint64_t nlo = lb + ((uint64_t)bstar << shift);
      const uint64_t w = (shift == 0) ? 0ull : ((1ull << shift) - 1ull);
      const uint64_t nhi = (kmax - nlo > w) ? nlo + w : kmax;
      __syncwarp();
      if (r == cnt) {  // the whole bucket and everything above it
        sel.thr = nlo;
        sel.kmin = U128{0ull, 0ull};
      } else if (cnt <= kListCap) {
        uint64_t* lbk = reinterpret_cast<uint64_t*>(hist + 256);
        uint32_t* lc = reinterpret_cast<uint32_t*>(lbk + kListCap);
        int base = 0;
        for (int m = 0; m < nslot; ++m) {
          bool ok;
          const uint64_t k = bkf(m, ok);
          const bool in = ok && k >= nlo && k <= nhi;
          const unsigned bal = __ballot_sync(0xffffffffu, in);
          if (in) {
            const int pos = base + __popc(bal & ((1u << lane) - 1u));
            lbk[pos] = k;
            lc[pos] = (uint32_t)(lane + 32 * m);
          }
          base += __popc(bal);
        }
        __syncwarp();
        auto lbkf = [&](int m, bool& ok) {
          const int q = lane + 32 * m;
          ok = q < cnt;
          return ok ? lbk[q] : 0ull;
        };
        auto lfullf = [&](int m) {
          uint32_t id;
          float vr, vc;
          hi_of((int)lc[lane + 32 * m], id, vr, vc);
          return cell_key(vr, vc, id);
        };
        sel = warp_select_top((cnt + 31) >> 5, lbkf, lfullf, r, nlo, hist);
      } else {
        sel = warp_select_top(nslot, bkf, fullf, K, lb, hist);
      }
    }
    // outputs in candidate order; gates = softmax over the K exact keys (hi part; the
    // TwoSum remainder is below 2^-53 relative)
    uint32_t id0;
    float r0, c0;
    const double k1v = hi_of(0, id0, r0, c0);
    float es = 0.f;
    int o = 0;
    const size_t ob = (size_t)th * K;
    for (int m = 0; m < nslot; ++m) {
      const int c = lane + 32 * m;
      uint32_t id = 0;
      float vr = 0.f, vc = 0.f;
      const double h = c < C ? hi_of(c, id, vr, vc) : 0.0;
      const uint64_t bk = c < C ? ord64(h) : 0ull;
      bool take = c < C && bk >= sel.thr;
      if (take && bk == sel.thr && (sel.kmin.hi | sel.kmin.lo)) take = ge(cell_key(vr, vc, id), sel.kmin);
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (take) {
        const int pos = o + __popc(bal & ((1u << lane) - 1u));
        const float e = expf((float)(h - k1v));
        es += e;
        idx[ob + pos] = (int32_t)id;
        gate[ob + pos] = e;
        if (score) score[ob + pos] = (float)(h - (double)lse_r - (double)lse_c);
      }
      o += __popc(bal);
    }
    const float inv = 1.0f / warp_sum(es);
    __syncwarp();
    for (int k = lane; k < K; k += 32) gate[ob + k] *= inv;
  }
}

// ---------------------------------------------------------------------------
// Ablation "w/o Cartesian Product Router": one 1024-thread CTA
// per token-head takes the exact top-K of its N dense logits by (value desc, id
// asc) -- radix select over the (value, ~id) keys, compaction, bitonic sort of the
// K survivors -- and writes ids and softmax gates in key order; score = s - lse.
__global__ void __launch_bounds__(1024)
    dense_select_kernel(int T, int N, int K, int plen, const float* __restrict__ logits, int32_t* __restrict__ idx,
                        float* __restrict__ gate, float* __restrict__ score) {
  extern __shared__ __align__(16) uint8_t smem[];
  SelShared<1024>& sh = *reinterpret_cast<SelShared<1024>*>(smem);
  uint64_t* sel = reinterpret_cast<uint64_t*>(smem + (sizeof(SelShared<1024>) + 15) / 16 * 16);
  for (int th = blockIdx.x; th < T; th += gridDim.x) {
    const float* lg = logits + (size_t)th * N;
    auto keyf = [lg](int i) { return half_key(lg[i], (uint32_t)i); };
    top_sorted<1024, uint64_t, 8>(N, K, keyf, sel, sh);
    const float mx = half_val(sel[0]);
    float es = 0.f;
    for (int k = threadIdx.x; k < K; k += 1024) es += expf(half_val(sel[k]) - mx);
    es = group_sum<1024>(es, sh);
    float lse = 0.f;
    if (score) {
      float s = 0.f;
      for (int i = threadIdx.x; i < N; i += 1024) s += __expf(lg[i] - mx);
      lse = mx + __logf(group_sum<1024>(s, sh));
    }
    for (int k = threadIdx.x; k < K; k += 1024) {
      const uint64_t q = sel[k];
      const size_t o = (size_t)th * K + k;
      idx[o] = (int32_t)half_idx(q);
      gate[o] = expf(half_val(q) - mx) / es;
      if (score) score[o] = half_val(q) - lse;
    }
    __syncthreads();
  }
  (void)plen;
}

}  // namespace

// host --------------------------------------------------------------------
omnimoe_status select_params(const omnimoe_dims& d, int64_t T, SelectParams* p, size_t* smem) {
  p->T = (int)T;
  p->n_rows = (int)d.n_rows;
  p->n_cols = (int)d.n_cols;
  p->top_k = (int)d.top_k;
  p->n_heads = (int)d.n_heads;
  const int64_t K1 = d.top_k + 1;
  p->kr1 = (int)std::min<int64_t>(K1, d.n_rows);
  p->kc1 = (int)std::min<int64_t>(K1, d.n_cols);
  int64_t C = 0;
  for (int64_t a = 1; a <= p->kr1; ++a) C += std::min<int64_t>(p->kc1, K1 / a);
  p->C = (int)C;
  // buffers hold max(sorted length, list length) keys (sort_len: the last key is the
  // radix-selected threshold and is not sorted)
  p->pkr = std::max(sort_len(p->kr1, p->n_rows), p->kr1);
  p->pkc = std::max(sort_len(p->kc1, p->n_cols), p->kc1);
  const int keep = (int)std::min<int64_t>(d.top_k, C);
  p->pkeep = std::max(sort_len(keep, (int)C), keep);
  p->sorted = 1;
  if (d.n_rows > 65535 || d.n_cols > 65535) {
    set_error("route: grid halves must be <= 65535");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  const size_t cand_bytes = ((size_t)C * 4 + 15) / 16 * 16;
  // one CTA per token-head: measured faster than one warp per token-head at K = 512
  // (the per-warp key buffers limit a warp-per-token-head kernel to 8 warps/SM);
  // small K uses select_warp_kernel instead (launch_select)
  // one CTA per token-head (1024 threads when K is in the thousands: the key buffers then
  // allow only one CTA per SM, and more threads hide more latency)
  p->group = tuning().select_warp_group && p->pkeep <= 1024 ? 32 : (p->pkeep >= 2048 ? 1024 : 256);
  const size_t gb = p->group == 32 ? group_bytes<32>(*p) : p->group == 256 ? group_bytes<256>(*p) : group_bytes<1024>(*p);
  p->groups_per_cta = p->group == 32 ? (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024 - cand_bytes) / gb)) : 1;
  *smem = cand_bytes + gb * p->groups_per_cta;
  if (*smem > 225 * 1024) {
    set_error("route: selection working set (" + std::to_string(*smem) +
              " bytes: K+1 sorted keys, both halves, " + std::to_string(C) +
              " product candidates) exceeds shared memory");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  return OMNIMOE_OK;
}

omnimoe_status launch_dense_select(const omnimoe_dims& d, int64_t T, const float* logits, int32_t* idx, float* gate,
                                   float* score, cudaStream_t st) {
  const int64_t N = d.n_rows * d.n_cols;
  const int K = (int)d.top_k;
  const int plen = std::max(sort_len(K, (int)N), K);
  const size_t sm = (sizeof(SelShared<1024>) + 15) / 16 * 16 + (size_t)plen * 8;
  if (sm > 200 * 1024) {
    set_error("dense router: K=" + std::to_string(K) + " sorted keys exceed shared memory");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (cudaFuncSetAttribute(dense_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
    set_error("dense router: cannot set shared memory");
    return OMNIMOE_ERR_CUDA;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dense_select_kernel, 1024, sm);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(T, (int64_t)num_sms() * std::max(per_sm, 1)));
  dense_select_kernel<<<grid, 1024, sm, st>>>((int)T, (int)N, K, plen, logits, idx, gate, score);
  OMNI_CHECK_LAUNCH("dense_select_kernel");
  return OMNIMOE_OK;
}

namespace {
int bucket_cand_count(int64_t K, int64_t n_rows, int64_t n_cols) {
  const int64_t kr = std::min(K, n_rows), kc = std::min(K, n_cols);
  int64_t C = 0;
  for (int64_t a = 0; a < kr; ++a) C += std::min(kc, K / (a + 1));
  return (int)C;
}
}  // namespace

size_t select_cand_ws_bytes(const omnimoe_dims& d) {
  return (size_t)bucket_cand_count(d.top_k, d.n_rows, d.n_cols) * 4;
}

omnimoe_status launch_select(const SelectParams& p, size_t smem, const float* logits, int32_t* idx,
                             float* gate, float* score, uint32_t* cand_ws, cudaStream_t st, const FusedRoute* fused) {
  if (p.top_k + 1 <= 32 && p.C <= 160) {  // small K: warp per token-head, repeated arg-max
    const int grid = std::max(1, std::min((p.T + 7) / 8, num_sms() * 8));
    const bool fz = fused && fused->kp > 0;
    select_warp_kernel<<<grid, 256, 0, st>>>(p, logits, idx, gate, score, fz ? fused->cand : nullptr,
                                             fz ? fused->part : nullptr, fz ? fused->kp : 0,
                                             std::max(1, p.n_heads), fz ? fused->counts : nullptr,
                                             fz ? fused->bad_x : nullptr);
    OMNI_CHECK_LAUNCH("select_warp_kernel");
    return OMNIMOE_OK;
  }
  if (!p.sorted && p.top_k >= 32 && std::min(p.top_k, p.n_rows) <= 1024 && std::min(p.top_k, p.n_cols) <= 1024 &&
      cand_ws &&
      !tuning().select_cta) {
    // candidate-order output (the layer path): warp per token-head, bucket selection
    const int K = p.top_k, kr = std::min(K, p.n_rows), kc = std::min(K, p.n_cols);
    const int C = bucket_cand_count(K, p.n_rows, p.n_cols);
    int Pr = 1, Pc = 1;
    while (Pr < kr) Pr <<= 1;
    while (Pc < kc) Pc <<= 1;
    const size_t per_warp = (size_t)(Pr + Pc) * 8 + 256 * 4 + kListCap * 12;
    const size_t cand_bytes = ((size_t)C * 4 + 15) / 16 * 16;
    int warps = 8;
    while (warps > 1 && warps * per_warp > 200 * 1024) warps >>= 1;
    // the candidate table: in shared memory when that still allows two CTAs per SM or
    // when one wave of one CTA per SM covers all token-heads (C4p: 0.51 vs 0.59 ms); else
    // in global memory, read through L1, for twice the resident warps (C4: 1.17 vs 1.49 ms)
    const bool fits = cand_bytes + warps * per_warp <= 200 * 1024;
    const bool in_smem =
        fits && (2 * (cand_bytes + warps * per_warp) <= 220 * 1024 || (int64_t)p.T <= (int64_t)warps * num_sms());
    const size_t sm = (in_smem ? cand_bytes : 0) + warps * per_warp;
    if (sm <= 200 * 1024) {
      cand_table_kernel<<<1, 1024, 0, st>>>(K, kr, kc, cand_ws);
      OMNI_CHECK_LAUNCH("cand_table_kernel");
      auto kern = in_smem ? select_bucket_kernel<true> : select_bucket_kernel<false>;
      if (!set_smem_attr((const void*)kern, (int)sm)) {
        set_error("route: cannot set select_bucket_kernel shared memory");
        return OMNIMOE_ERR_CUDA;
      }
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, sm);
      const int grid = std::max(1, std::min((p.T + warps - 1) / warps, num_sms() * std::max(per_sm, 1)));
      kern<<<grid, warps * 32, sm, st>>>(p, C, Pr, Pc, cand_ws, logits, idx, gate, score);
      OMNI_CHECK_LAUNCH("select_bucket_kernel");
      return OMNIMOE_OK;
    }
  }
  auto kern = p.group == 32 ? select_kernel<32> : p.group == 256 ? select_kernel<256> : select_kernel<1024>;
  const int threads = p.group == 32 ? 32 * p.groups_per_cta : p.group;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("route: cannot set select_kernel shared memory");
    return OMNIMOE_ERR_CUDA;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  const int per_cta = threads / p.group;
  const int grid = std::max(1, std::min((p.T + per_cta - 1) / per_cta, num_sms() * std::max(per_sm, 1)));
  kern<<<grid, threads, smem, st>>>(p, logits, idx, gate, score);
  OMNI_CHECK_LAUNCH("select_kernel");
  return OMNIMOE_OK;
}

}  // namespace omni
