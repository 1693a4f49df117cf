// Cartesian Product Router kernels, steps a1-a3 of DESIGN.md.
//
//  canon_logits_kernel   canonical logits: fp64 FMA over k in index order, one
//                        rounding to fp32 (reading Q9).  Used for every token-head
//                        in canonical mode and for flagged token-heads in fast mode.
//  select_kernel         one CTA per token-head: per-half sort by (value desc,
//                        index asc) + logsumexp (Eq.LSM); exact product candidates
//                        (a*b <= K+1) with TwoSum keys; CTA bitonic sort of the
//                        candidates; gates = softmax over the selected keys
//                        (Eq.Gate); K/K+1 gap certification.
#include "router.cuh"

namespace omni {
namespace {

constexpr int kSelThreads = 512;

// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }

// grid: full mode blockIdx over T*nrb; list mode persistent over list entries.
template <typename T>
__global__ void __launch_bounds__(128)
    canon_logits_kernel(const T* __restrict__ x, const T* __restrict__ sub, int d, int h, int R,
                        float* __restrict__ logits, int T_total, const int32_t* __restrict__ list,
                        const int32_t* __restrict__ list_count) {
  __shared__ float st[128][33];
  __shared__ double xs[32];
  const int nrb = (R + 127) / 128;
  const int total = list ? (*list_count) * nrb : T_total * nrb;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int th = list ? list[item / nrb] : item / nrb;
    const int rb = item % nrb;
    const int l = th / h, hh = th % h;
    const T* xl = x + (size_t)l * d;
    const int r0 = rb * 128;
    const int r = r0 + threadIdx.x;
    double acc = 0.0;
    for (int k0 = 0; k0 < d; k0 += 32) {
      __syncthreads();
      if (threadIdx.x < 32) xs[threadIdx.x] = (k0 + threadIdx.x < d) ? (double)to_f(xl[k0 + threadIdx.x]) : 0.0;
      for (int i = threadIdx.x; i < 128 * 32; i += 128) {
        int rr = i / 32, kk = i % 32;
        int gr = r0 + rr, gk = k0 + kk;
        st[rr][kk] = (gr < R && gk < d) ? to_f(sub[((size_t)hh * R + gr) * d + gk]) : 0.f;
      }
      __syncthreads();
      const int kmax = min(32, d - k0);
      for (int kk = 0; kk < kmax; ++kk) acc = fma(xs[kk], (double)st[threadIdx.x][kk], acc);
    }
    if (r < R) logits[(size_t)th * R + r] = (float)acc;
  }
}

// ---------------------------------------------------------------------------
struct Key128 {
  uint64_t a, b;  // a = ord64(hi), b = ord32(lo) << 32 | (0xFFFFFFFF - flat id)
};
__device__ __forceinline__ bool gt128(const Key128& x, const Key128& y) {
  return x.a > y.a || (x.a == y.a && x.b > y.b);
}

template <class K, class G>
__device__ void bitonic_desc(K* a, int n, G greater) {
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = (lo & size) == 0;
        K p = a[lo], q = a[hi];
        if (desc ? greater(q, p) : greater(p, q)) {
          a[lo] = q;
          a[hi] = p;
        }
      }
    }
  __syncthreads();
}

// deterministic block reductions (fixed tree)
__device__ float block_max(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < nw; ++i) r = fmaxf(r, red[i]);
  return r;
}
__device__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float r = 0.f;
  for (int i = 0; i < nw; ++i) r += red[i];
  return r;
}

__device__ __forceinline__ uint64_t half_key(float v, uint32_t i) {
  v = v + 0.0f;  // canonicalise -0.0 -> +0.0 so equal values compare equal
  return ((uint64_t)ord32(v) << 32) | (uint64_t)(0xFFFFFFFFu - i);
}

__global__ void __launch_bounds__(kSelThreads)
    select_kernel(SelectParams p, const float* __restrict__ logits, int32_t* __restrict__ idx,
                  float* __restrict__ gate, float* __restrict__ score, int32_t* __restrict__ flag_list,
                  int32_t* __restrict__ flag_count, const int32_t* __restrict__ list,
                  const int32_t* __restrict__ list_count) {
  extern __shared__ __align__(16) uint8_t sm[];
  Key128* cand = reinterpret_cast<Key128*>(sm);
  uint64_t* kr = reinterpret_cast<uint64_t*>(cand + p.pc);
  uint64_t* kc = kr + p.pr;
  int32_t* P = reinterpret_cast<int32_t*>(kc + p.pcol);
  float* red = reinterpret_cast<float*>(P + p.kr1 + 1);

  const int R = p.n_rows + p.n_cols;
  const int K1 = p.top_k + 1;
  // P[a] = number of candidates with (0-based) row rank < a; the same for every
  // token-head, so computed once per CTA (rows a+1 admit min(kc1, (K+1)/(a+1)) columns)
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int a = 0; a < p.kr1; ++a) {
      P[a] = acc;
      acc += min(p.kc1, K1 / (a + 1));
    }
    P[p.kr1] = acc;
  }
  __syncthreads();
  const int C = P[p.kr1];
  const int total = list ? *list_count : p.T;
  for (int item = blockIdx.x; item < total; item += gridDim.x) {
    const int th = list ? list[item] : item;
    const float* lg = logits + (size_t)th * R;
    // ---- a2: load halves as sortable keys; logsumexp per half (Eq.LSM) ----
    float mr = -INFINITY, mc = -INFINITY;
    for (int i = threadIdx.x; i < p.pr; i += blockDim.x) {
      float v = i < p.n_rows ? lg[i] : -INFINITY;
      kr[i] = i < p.n_rows ? half_key(v, i) : 0ull;
      mr = fmaxf(mr, v);
    }
    for (int i = threadIdx.x; i < p.pcol; i += blockDim.x) {
      float v = i < p.n_cols ? lg[p.n_rows + i] : -INFINITY;
      kc[i] = i < p.n_cols ? half_key(v, i) : 0ull;
      mc = fmaxf(mc, v);
    }
    mr = block_max(mr, red);
    mc = block_max(mc, red);
    float sr_ = 0.f, sc_ = 0.f;
    for (int i = threadIdx.x; i < p.n_rows; i += blockDim.x) sr_ += __expf(lg[i] - mr);
    for (int i = threadIdx.x; i < p.n_cols; i += blockDim.x) sc_ += __expf(lg[p.n_rows + i] - mc);
    const float lse_r = mr + __logf(block_sum(sr_, red));
    const float lse_c = mc + __logf(block_sum(sc_, red));
    auto g64 = [](uint64_t x, uint64_t y) { return x > y; };
    bitonic_desc(kr, p.pr, g64);
    bitonic_desc(kc, p.pcol, g64);
    // ---- a3: candidate ranks (a, b), 1-based, with a*b <= K+1 ----
    for (int c = threadIdx.x; c < p.pc; c += blockDim.x) {
      Key128 k{0ull, 0ull};
      if (c < C) {
        int lo = 0, hi = p.kr1 - 1;  // largest a with P[a] <= c
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (P[mid] <= c) lo = mid; else hi = mid - 1;
        }
        const int a = lo, b = c - P[a];
        const uint64_t ka = kr[a], kb = kc[b];
        const float va = ord32_inv((uint32_t)(ka >> 32)), vb = ord32_inv((uint32_t)(kb >> 32));
        const uint32_t ia = 0xFFFFFFFFu - (uint32_t)ka, ib = 0xFFFFFFFFu - (uint32_t)kb;
        // exact key: TwoSum in fp64 (hi, lo); lo is exactly representable in fp32
        const double da = (double)va, db = (double)vb;
        double s = da + db;
        const double bb = s - da;
        double e = (da - (s - bb)) + (db - bb);
        s = s + 0.0;
        const float ef = (float)e + 0.0f;
        const uint32_t n = ia * (uint32_t)p.n_cols + ib;
        k.a = ord64(s);
        k.b = ((uint64_t)ord32(ef) << 32) | (uint64_t)(0xFFFFFFFFu - n);
      }
      cand[c] = k;
    }
    bitonic_desc(cand, p.pc, [](const Key128& x, const Key128& y) { return gt128(x, y); });
    // ---- gates (Eq.Gate): softmax over the K selected exact keys ----
    const Key128 top = cand[0];
    const double hi1 = __longlong_as_double((long long)((top.a & 0x8000000000000000ull) ? (top.a & 0x7FFFFFFFFFFFFFFFull) : ~top.a));
    const float lo1 = ord32_inv((uint32_t)(top.b >> 32));
    float esum = 0.f;
    for (int k = threadIdx.x; k < p.top_k; k += blockDim.x) {
      const Key128 q = cand[k];
      const double hk = __longlong_as_double((long long)((q.a & 0x8000000000000000ull) ? (q.a & 0x7FFFFFFFFFFFFFFFull) : ~q.a));
      const float lk = ord32_inv((uint32_t)(q.b >> 32));
      esum += expf((float)((hk - hi1) + (double)(lk - lo1)));
    }
    esum = block_sum(esum, red);
    const float inv = 1.0f / esum;
    for (int k = threadIdx.x; k < p.top_k; k += blockDim.x) {
      const Key128 q = cand[k];
      const double hk = __longlong_as_double((long long)((q.a & 0x8000000000000000ull) ? (q.a & 0x7FFFFFFFFFFFFFFFull) : ~q.a));
      const float lk = ord32_inv((uint32_t)(q.b >> 32));
      const size_t o = (size_t)th * p.top_k + k;
      idx[o] = (int32_t)(0xFFFFFFFFu - (uint32_t)q.b);
      gate[o] = expf((float)((hk - hi1) + (double)(lk - lo1))) * inv;
      if (score) score[o] = (float)(hk + (double)lk - (double)lse_r - (double)lse_c);
    }
    // ---- certification of fast logits ----
    if (threadIdx.x == 0 && p.cert_eps > 0.f && C > p.top_k) {
      const Key128 qk = cand[p.top_k - 1], qn = cand[p.top_k];
      const double hk = __longlong_as_double((long long)((qk.a & 0x8000000000000000ull) ? (qk.a & 0x7FFFFFFFFFFFFFFFull) : ~qk.a));
      const double hn = __longlong_as_double((long long)((qn.a & 0x8000000000000000ull) ? (qn.a & 0x7FFFFFFFFFFFFFFFull) : ~qn.a));
      const double gap = (hk - hn) + (double)(ord32_inv((uint32_t)(qk.b >> 32)) - ord32_inv((uint32_t)(qn.b >> 32)));
      if (gap <= 4.0 * (double)p.cert_eps) flag_list[atomicAdd(flag_count, 1)] = th;
    }
    __syncthreads();
  }
}

int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace

// host --------------------------------------------------------------------
omnimoe_status select_params(const omnimoe_dims& d, int64_t T, SelectParams* p, size_t* smem) {
  p->T = (int)T;
  p->n_rows = (int)d.n_rows;
  p->n_cols = (int)d.n_cols;
  p->top_k = (int)d.top_k;
  const int K1 = p->top_k + 1;
  p->kr1 = (int)std::min<int64_t>(K1, d.n_rows);
  p->kc1 = (int)std::min<int64_t>(K1, d.n_cols);
  int64_t C = 0;
  for (int a = 1; a <= p->kr1; ++a) C += std::min<int64_t>(p->kc1, K1 / a);
  p->pr = pow2ceil(p->n_rows);
  p->pcol = pow2ceil(p->n_cols);
  p->pc = pow2ceil((int)std::max<int64_t>(C, 2));
  if (p->pr > 8192 || p->pcol > 8192 || p->pc > 8192) {
    set_error("route: grid halves must be <= 8192 and product candidates (a*b <= K+1) <= 8192; got " +
              std::to_string(C) + " candidates");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  *smem = (size_t)p->pc * sizeof(Key128) + (size_t)(p->pr + p->pcol) * 8 + (size_t)(p->kr1 + 1) * 4 + 64 * 4 + 64;
  if (*smem > 227 * 1024) {
    set_error("route: selection working set exceeds shared memory");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  return OMNIMOE_OK;
}

omnimoe_status launch_select(const SelectParams& p, size_t smem, const float* logits, int32_t* idx,
                             float* gate, float* score, int32_t* flag_list, int32_t* flag_count,
                             const int32_t* list, const int32_t* list_count, cudaStream_t st) {
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel, kSelThreads, smem);
  int grid = std::min(p.T, kSMs * std::max(per_sm, 1));
  if (grid <= 0) return OMNIMOE_OK;
  select_kernel<<<grid, kSelThreads, smem, st>>>(p, logits, idx, gate, score, flag_list, flag_count,
                                                 list, list_count);
  OMNI_CHECK_LAUNCH("select_kernel");
  return OMNIMOE_OK;
}

omnimoe_status launch_canon_logits(int dtype, const void* x, const void* sub, int d, int h, int R,
                                   float* logits, int T, const int32_t* list,
                                   const int32_t* list_count, cudaStream_t st) {
  const int nrb = (R + 127) / 128;
  int grid = list ? std::min(T * nrb, kSMs * 8) : T * nrb;
  if (grid <= 0) return OMNIMOE_OK;
  if (dtype == OMNIMOE_BF16)
    canon_logits_kernel<__nv_bfloat16><<<grid, 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(sub), d, h, R,
        logits, T, list, list_count);
  else
    canon_logits_kernel<float><<<grid, 128, 0, st>>>(static_cast<const float*>(x),
                                                     static_cast<const float*>(sub), d, h, R,
                                                     logits, T, list, list_count);
  OMNI_CHECK_LAUNCH("canon_logits_kernel");
  return OMNIMOE_OK;
}

}  // namespace omni
