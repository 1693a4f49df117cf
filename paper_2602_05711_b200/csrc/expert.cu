// Grouped atomic-expert compute + scatter-add (Eq.Grouped), step
// a6 of DESIGN.md.
//
//  expert_warp_kernel   plan with B = 1 (expert-major): one warp owns one active
//                       expert at a time, holds its w_e / v_e rows in registers
//                       (read from HBM exactly once per layer, D_expert =
//                       2d|E_active|), then streams the expert's
//                       tasks in ascending token order: gather x_l,
//                       z = x_l . w_e in fp32, a = g * sigma(z), scatter-add
//                       a * v_e into y_routed[l] with red.global.add.v4.f32.
//  expert_group_kernel  plan with B > 1, sorted by (group q, token l) (Eq.Sort):
//                       one warp per run (q, l): x_l and an fp32 partial y_l live
//                       in registers while the warp walks the run's experts
//                       (w_e, v_e streamed; runs are taken in plan order, so the
//                       warps in flight cover a window of ~1 group whose rows
//                       stay L2-resident after one HBM read), then ONE red.v4
//                       scatter per run instead of one per task.
#include <cmath>
#include <cstdlib>
#include <string>

#include "schedule.cuh"
#include "tcgen05.cuh"

namespace omni {
namespace {


template <typename T>
struct VecT;
template <>
struct VecT<__nv_bfloat16> {
  static constexpr int E = 8;  // elements per 16-byte vector
  __device__ static __forceinline__ void unpack(const uint4& u, float (&f)[8]) {
    f[0] = bf16_lo(u.x); f[1] = bf16_hi(u.x); f[2] = bf16_lo(u.y); f[3] = bf16_hi(u.y);
    f[4] = bf16_lo(u.z); f[5] = bf16_hi(u.z); f[6] = bf16_lo(u.w); f[7] = bf16_hi(u.w);
  }
};
template <>
struct VecT<float> {
  static constexpr int E = 4;
  __device__ static __forceinline__ void unpack(const uint4& u, float (&f)[4]) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};

__device__ __forceinline__ uint4 ld_stream(const void* p) {  // read-once rows: no L1 allocation
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_vec(const void* p) {
  return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

template <typename T, int NV>
__global__ void __launch_bounds__(256)
    expert_warp_kernel(int d, const T* __restrict__ x, const T* __restrict__ W,
                       const T* __restrict__ V, const int32_t* __restrict__ offsets,
                       const int32_t* __restrict__ active, const int32_t* __restrict__ n_active,
                       const int32_t* __restrict__ stok, const float* __restrict__ sgate,
                       float* __restrict__ y, int act) {
  constexpr int E = VecT<T>::E;
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * (int64_t)blockDim.x) >> 5);
  const int na = *n_active;
  for (int tau = gw; tau < na; tau += nw) {
    const int e = active[tau];
    const int beg = offsets[e], end = offsets[e + 1];
    uint4 wv[NV], vv[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * E;
      if (c < d) {
        wv[j] = ld_stream(W + (size_t)e * d + c);
        vv[j] = ld_stream(V + (size_t)e * d + c);
      } else {
        wv[j] = make_uint4(0, 0, 0, 0);
        vv[j] = make_uint4(0, 0, 0, 0);
      }
    }
    for (int p = beg; p < end; ++p) {
      const int l = stok[p];
      const float g = sgate[p];
      const T* xl = x + (size_t)l * d;
      uint4 xv[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * E;
        xv[j] = c < d ? ld_vec(xl + c) : make_uint4(0, 0, 0, 0);
      }
      float z = 0.f;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        float xf[E], wf[E];
        VecT<T>::unpack(xv[j], xf);
        VecT<T>::unpack(wv[j], wf);
#pragma unroll
        for (int i = 0; i < E; ++i) z = fmaf(xf[i], wf[i], z);
      }
      z = warp_sum(z);
      const float a = g * (act == OMNIMOE_IDENTITY ? z : silu_f(z));
      float* yl = y + (size_t)l * d;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * E;
        if (c < d) {
          float vf[E];
          VecT<T>::unpack(vv[j], vf);
#pragma unroll
          for (int i = 0; i < E; i += 4) red_add_v4(yl + c + i, a * vf[i], a * vf[i + 1], a * vf[i + 2], a * vf[i + 3]);
        }
      }
    }
  }
}

template <typename T, int NV>
__global__ void __launch_bounds__(256)
    expert_group_kernel(int d, const T* __restrict__ x, const T* __restrict__ W,
                        const T* __restrict__ V, const int32_t* __restrict__ run_off,
                        const int32_t* __restrict__ n_runs_p, const int32_t* __restrict__ m_loc_p,
                        const int32_t* __restrict__ stok, const int32_t* __restrict__ sexp,
                        const float* __restrict__ sgate, float* __restrict__ y, int act,
                        int* __restrict__ work) {
  constexpr int E = VecT<T>::E;
  constexpr int kChunk = 4;  // runs claimed per atomic
  const int lane = threadIdx.x & 31;
  const int n_runs = *n_runs_p, m_loc = *m_loc_p;
  // runs are claimed in plan order through one counter, so the warps in flight
  // always cover a narrow window of groups (their W/V rows stay L2-resident)
  int r0 = 0;
  if (lane == 0) r0 = atomicAdd(work, kChunk);
  r0 = __shfl_sync(0xffffffffu, r0, 0);
  for (int r = r0; r < n_runs;) {
    const int beg = run_off[r];
    const int end = r + 1 < n_runs ? run_off[r + 1] : m_loc;
    const int l = stok[beg];
    const T* xl = x + (size_t)l * d;
    uint4 xv[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * E;
      xv[j] = c < d ? ld_vec(xl + c) : make_uint4(0, 0, 0, 0);
    }
    float acc[NV][E];
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (int i = 0; i < E; ++i) acc[j][i] = 0.f;
    for (int p0 = beg; p0 < end; p0 += 32) {
      // the next (up to) 32 tasks' expert ids and gates, one per lane
      const int pl = p0 + lane;
      const int e_l = pl < end ? sexp[pl] : 0;
      const float g_l = pl < end ? sgate[pl] : 0.f;
      const int cnt = min(32, end - p0);
      for (int t = 0; t < cnt; ++t) {
        const int e = __shfl_sync(0xffffffffu, e_l, t);
        const float g = __shfl_sync(0xffffffffu, g_l, t);
        const T* we = W + (size_t)e * d;
        const T* ve = V + (size_t)e * d;
        uint4 wv[NV], vv[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const int c = (j * 32 + lane) * E;
          wv[j] = c < d ? ld_vec(we + c) : make_uint4(0, 0, 0, 0);
          vv[j] = c < d ? ld_vec(ve + c) : make_uint4(0, 0, 0, 0);
        }
        float z = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          float xf[E], wf[E];
          VecT<T>::unpack(xv[j], xf);
          VecT<T>::unpack(wv[j], wf);
#pragma unroll
          for (int i = 0; i < E; ++i) z = fmaf(xf[i], wf[i], z);
        }
        z = warp_sum(z);
        const float a = g * (act == OMNIMOE_IDENTITY ? z : silu_f(z));
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          float vf[E];
          VecT<T>::unpack(vv[j], vf);
#pragma unroll
          for (int i = 0; i < E; ++i) acc[j][i] = fmaf(a, vf[i], acc[j][i]);
        }
      }
    }
    float* yl = y + (size_t)l * d;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * E;
      if (c < d) {
#pragma unroll
        for (int i = 0; i < E; i += 4) red_add_v4(yl + c + i, acc[j][i], acc[j][i + 1], acc[j][i + 2], acc[j][i + 3]);
      }
    }
    if (++r == r0 + kChunk) {
      if (lane == 0) r0 = atomicAdd(work, kChunk);
      r = r0 = __shfl_sync(0xffffffffu, r0, 0);
    }
  }
}

// ---- packed math helpers (sm_100a) ----
// z += x.lo*w.lo + x.hi*w.hi with bf16 inputs and fp32 accumulation (FHFMA.BF16)
__device__ __forceinline__ float dot2_bf16(float z, uint32_t xp, uint32_t wp) {
  asm("{ .reg .b16 xl, xh, wl, wh;\n\t"
      "mov.b32 {xl, xh}, %1;\n\t"
      "mov.b32 {wl, wh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, xl, wl, %0;\n\t"
      "fma.rn.f32.bf16 %0, xh, wh, %0; }"
      : "+f"(z)
      : "r"(xp), "r"(wp));
  return z;
}
// acc.{x,y} += a * {v.lo, v.hi} (bf16x2 v widened exactly to fp32) with one FFMA2
__device__ __forceinline__ void axpy2_bf16(unsigned long long& acc, unsigned long long a2, uint32_t vp) {
  const unsigned long long v2 = ((unsigned long long)(vp & 0xFFFF0000u) << 32) | (unsigned long long)(vp << 16);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a2), "l"(v2));
}
// lo += a * bf16(vp.lo), hi += a * bf16(vp.hi): fma.rn.f32.bf16 on the halves of vp (FHFMA)
__device__ __forceinline__ void fma_bf16_pair(float& lo, float& hi, unsigned short a, uint32_t vp) {
  asm("{ .reg .b16 vl, vh;\n\t"
      "mov.b32 {vl, vh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, %3, vl, %0;\n\t"
      "fma.rn.f32.bf16 %1, %3, vh, %1; }"
      : "+f"(lo), "+f"(hi)
      : "r"(vp), "h"(a));
}
__device__ __forceinline__ float lo_f(unsigned long long p) { return __uint_as_float((uint32_t)p); }
__device__ __forceinline__ float hi_f(unsigned long long p) { return __uint_as_float((uint32_t)(p >> 32)); }

// ---------------------------------------------------------------------------
// expert_group_tma_kernel: the run-major executor with its expert rows staged by
// the TMA engine.  Each warp is independent: lane 0 is its producer, issuing
// 1-D cp.async.bulk copies of w_e, v_e (and x_l at the first task of a run) into
// an S-deep ring of shared-memory stages completed on per-stage mbarriers; all
// 32 lanes consume stage by stage (x_l held as fp32 in registers for the whole
// run, dot product from shared memory, shuffle reduce, fp32 axpy into the run's
// register accumulator), one red.v4 scatter per run.  Rows are in flight S-1
// tasks ahead of the math, independent of the warp count.
constexpr int kGChunk = 4;  // runs claimed per atomic

struct StageMeta {
  float g;
  int tok;
  int flags;  // 1: first task of its run, 2: last task of its run, 4: last task of its chunk
  int pad;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// same, with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void red_add_v4_hint(float* p, float a, float b, float c, float d, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint4 ld_vec_hint(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

template <int NV, int S>
__global__ void __launch_bounds__(256, 1)
    expert_group_tma_kernel(int d, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ W,
                            const __nv_bfloat16* __restrict__ V, const int32_t* __restrict__ run_off,
                            const int32_t* __restrict__ n_runs_p, const int32_t* __restrict__ m_loc_p,
                            const int32_t* __restrict__ stok, const int32_t* __restrict__ sexp,
                            const float* __restrict__ sgate, float* __restrict__ y, int act,
                            int* __restrict__ work, int hints) {
  extern __shared__ __align__(128) uint8_t smem[];
  // L2 eviction priorities (hints bit 0: W/V evict_first, 1: y_routed evict_last,
  // 2: x evict_last, 3: W/V evict_last)
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
  const bool wv_hint = hints & 9, y_hint = hints & 2, x_hint = hints & 4;
  const uint64_t pol = (hints & 1) ? pol_first : pol_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t row_bytes = (uint32_t)d * 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);                    // [nwarps][S]
  StageMeta* metas = reinterpret_cast<StageMeta*>(bars + nwarps * S);    // [nwarps][S]
  uint8_t* rows = reinterpret_cast<uint8_t*>(metas + nwarps * S);
  rows = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(rows) + 127) & ~uintptr_t(127));
  uint64_t* bar = bars + wid * S;
  StageMeta* meta = metas + wid * S;
  uint8_t* ring = rows + (size_t)wid * S * 2 * row_bytes;  // stage s: w_e | v_e
  if (lane == 0) {
    for (int s = 0; s < S; ++s) tc::mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int n_runs = *n_runs_p, m_loc = *m_loc_p;
  // two-slot queue of claimed chunks; bnd[s]: lane i holds the first task of run r0+i
  int nr[2], bnd[2];
  auto claim = [&](int slot) {
    int r = 0;
    if (lane == 0) r = atomicAdd(work, kGChunk);
    r = __shfl_sync(0xffffffffu, r, 0);
    const int n = max(0, min(kGChunk, n_runs - r));
    const int b = (lane <= n && n > 0) ? (r + lane < n_runs ? run_off[r + lane] : m_loc) : 0;
    if (slot) { nr[1] = n; bnd[1] = b; } else { nr[0] = n; bnd[0] = b; }
  };
  auto bound = [&](int slot, int i) { return __shfl_sync(0xffffffffu, slot ? bnd[1] : bnd[0], i); };
  claim(0);
  nr[1] = 0;
  bnd[1] = 0;
  // producer cursor: chunk slot ps, run prun inside it, task ppos in [.., pend)
  int ps = 0, prun = 0, ppos = 0, pend = 0;
  bool pdone = nr[0] == 0, pstart = true;
  if (!pdone) {
    ppos = bound(0, 0);
    pend = bound(0, 1);
  }
  int cs = 0;  // consumer chunk slot
  uint32_t pn = 0, cn = 0;
  int wb = -64, we = 0, wt = 0;   // task metadata window [wb, wb + 32): lane i holds task wb + i
  float wg = 0.f;
  uint4 xv[NV];                   // x_l of the current run (packed bf16)
  unsigned long long acc[NV][4];  // fp32 pairs of the run's partial y_l
  uint4 xnext[NV];                // x row of the next run to start, loaded ahead
  int xnext_tok = -1;
#pragma unroll
  for (int j = 0; j < NV; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[j][i] = 0ull;

  while (true) {
    // ---- producer: keep S tasks in flight ----
    while (!pdone && pn < cn + S) {
      if (ppos == pend) {  // next run (and chunk)
        const int nrun = prun + 1;
        if (nrun == (ps ? nr[1] : nr[0])) {
          if (cs != ps) break;  // the consumer still drains the other slot: retry later
          ps ^= 1;
          claim(ps);
          prun = 0;
          if ((ps ? nr[1] : nr[0]) == 0) {
            pdone = true;
            break;
          }
        } else {
          prun = nrun;
        }
        ppos = bound(ps, prun);
        pend = bound(ps, prun + 1);
        pstart = true;
      }
      const int s = pn % S;
      if (ppos < wb || ppos >= wb + 32) {  // refill the metadata window: 32 tasks, one per lane
        wb = ppos;
        const int q = wb + lane;
        we = q < m_loc ? sexp[q] : 0;
        wg = q < m_loc ? sgate[q] : 0.f;
        wt = q < m_loc ? stok[q] : 0;
      }
      const int e = __shfl_sync(0xffffffffu, we, ppos - wb);
      const float mg = __shfl_sync(0xffffffffu, wg, ppos - wb);
      const int mt = __shfl_sync(0xffffffffu, wt, ppos - wb);
      if (lane == 0) {
        StageMeta m;
        m.g = mg;
        m.tok = mt;
        const bool last_run = ppos + 1 == pend;
        m.flags = (pstart ? 1 : 0) | (last_run ? 2 : 0) |
                  ((last_run && prun + 1 == (ps ? nr[1] : nr[0])) ? 4 : 0);
        meta[s] = m;
        uint8_t* st = ring + (size_t)s * 2 * row_bytes;
        tc::mbar_expect_tx(&bar[s], 2u * row_bytes);
        if (wv_hint) {
          bulk_g2s_hint(st, W + (size_t)e * d, row_bytes, &bar[s], pol);
          bulk_g2s_hint(st + row_bytes, V + (size_t)e * d, row_bytes, &bar[s], pol);
        } else {
          bulk_g2s(st, W + (size_t)e * d, row_bytes, &bar[s]);
          bulk_g2s(st + row_bytes, V + (size_t)e * d, row_bytes, &bar[s]);
        }
      }
      pstart = false;
      ++ppos;
      ++pn;
    }
    if (cn == pn) break;  // nothing in flight and nothing more to issue
    __syncwarp();  // lane 0's meta stores are visible to the whole warp
    // ---- consumer: task cn ----
    const int s = cn % S;
    tc::mbar_wait(&bar[s], (cn / S) & 1);
    const StageMeta m = meta[s];
    const uint8_t* st = ring + (size_t)s * 2 * row_bytes;
    if (m.flags & 1) {  // first task of a run: x_l into registers (prefetched if possible)
      if (xnext_tok != m.tok) {
#pragma unroll
        for (int j = 0; j < NV; ++j)
          xnext[j] = x_hint ? ld_vec_hint(x + (size_t)m.tok * d + (j * 32 + lane) * 8, pol_last)
                            : ld_vec(x + (size_t)m.tok * d + (j * 32 + lane) * 8);
      }
#pragma unroll
      for (int j = 0; j < NV; ++j) xv[j] = xnext[j];
      xnext_tok = -1;
    }
    // prefetch the x row of the next run that starts inside the ring
    if (xnext_tok < 0) {
      for (uint32_t q = cn + 1; q < pn; ++q) {
        const StageMeta& mq = meta[q % S];
        if (mq.flags & 1) {
          xnext_tok = mq.tok;
#pragma unroll
          for (int j = 0; j < NV; ++j)
            xnext[j] = x_hint ? ld_vec_hint(x + (size_t)xnext_tok * d + (j * 32 + lane) * 8, pol_last)
                              : ld_vec(x + (size_t)xnext_tok * d + (j * 32 + lane) * 8);
          break;
        }
      }
    }
    // z = x_l . w_e: FHFMA.BF16 into NV independent partial sums
    float zp[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const uint4 u = *reinterpret_cast<const uint4*>(st + (size_t)(j * 32 + lane) * 16);
      float t = dot2_bf16(0.f, xv[j].x, u.x);
      t = dot2_bf16(t, xv[j].y, u.y);
      t = dot2_bf16(t, xv[j].z, u.z);
      zp[j] = dot2_bf16(t, xv[j].w, u.w);
    }
    float z = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) z += zp[j];
    z = warp_sum(z);
    const float a = m.g * (act == OMNIMOE_IDENTITY ? z : silu_f(z));
    const unsigned long long a2 = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const uint4 u = *reinterpret_cast<const uint4*>(st + row_bytes + (size_t)(j * 32 + lane) * 16);
      axpy2_bf16(acc[j][0], a2, u.x);
      axpy2_bf16(acc[j][1], a2, u.y);
      axpy2_bf16(acc[j][2], a2, u.z);
      axpy2_bf16(acc[j][3], a2, u.w);
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // stage s may be refilled now
    if (m.flags & 2) {
      float* yl = y + (size_t)m.tok * d;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * 8;
        if (y_hint) {
          red_add_v4_hint(yl + c, lo_f(acc[j][0]), hi_f(acc[j][0]), lo_f(acc[j][1]), hi_f(acc[j][1]), pol_last);
          red_add_v4_hint(yl + c + 4, lo_f(acc[j][2]), hi_f(acc[j][2]), lo_f(acc[j][3]), hi_f(acc[j][3]), pol_last);
        } else {
          red_add_v4(yl + c, lo_f(acc[j][0]), hi_f(acc[j][0]), lo_f(acc[j][1]), hi_f(acc[j][1]));
          red_add_v4(yl + c + 4, lo_f(acc[j][2]), hi_f(acc[j][2]), lo_f(acc[j][3]), hi_f(acc[j][3]));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] = 0ull;
      }
    }
    if (m.flags & 4) cs ^= 1;
    ++cn;
  }
}

template <int NV, int S>
omnimoe_status launch_group_tma(int d, const void* x, const void* W, const void* V, const omnimoe_plan& plan,
                                const int32_t* m_loc, float* y, int act, int* work, cudaStream_t st) {
  const size_t per_warp = (size_t)S * 2 * d * 2;
  const int warps = (int)std::min<size_t>(8, (size_t)(200 * 1024) / per_warp);
  const size_t smem = 128 + (size_t)warps * S * (8 + sizeof(StageMeta)) + (size_t)warps * per_warp + 128;
  auto kern = expert_group_tma_kernel<NV, S>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    set_error("expert_fwd: cannot set shared memory of the TMA group kernel");
    return OMNIMOE_ERR_CUDA;
  }
  kern<<<num_sms(), warps * 32, smem, st>>>(d, static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(W),
                                       static_cast<const __nv_bfloat16*>(V), plan.run_offsets, plan.n_runs, m_loc,
                                       plan.sorted_token, plan.sorted_expert, plan.sorted_gate, y, act, work,
                                       tuning().l2_hints);
  OMNI_CHECK_LAUNCH("expert_group_tma_kernel");
  return OMNIMOE_OK;
}

// ---------------------------------------------------------------------------
// expert_token_kernel: the token-centric execution the paper ablates ("w/o ECS",
// PAPER:241, 253, 396; Fig. 4a): one warp per token walks its h*K routed experts in
// routing order, gathering w_e and v_e from HBM for every task (no reuse across
// tokens), z = x_l . w_e, y_l += g * sigma(z) * v_e in registers; y_routed[l] is
// written once (no atomics).  Same arithmetic as the grouped kernels.
template <int NV>
__global__ void __launch_bounds__(256)
    expert_token_kernel(int d, int64_t L, int hk, const __nv_bfloat16* __restrict__ x,
                        const __nv_bfloat16* __restrict__ W, const __nv_bfloat16* __restrict__ V,
                        const int32_t* __restrict__ idx, const float* __restrict__ gate, int64_t begin,
                        int64_t end, float* __restrict__ y, int accumulate, int act) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t l = gw; l < L; l += nw) {
    uint4 xv[NV];
    unsigned long long acc[NV][4];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      xv[j] = ld_vec(x + (size_t)l * d + (j * 32 + lane) * 8);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[j][i] = 0ull;
    }
    for (int k0 = 0; k0 < hk; k0 += 32) {
      const int kk = k0 + lane;
      const int n_l = kk < hk ? idx[l * hk + kk] : -1;
      const float g_l = kk < hk ? gate[l * hk + kk] : 0.f;
      const int cnt = min(32, hk - k0);
      for (int t = 0; t < cnt; ++t) {
        const int n = __shfl_sync(0xffffffffu, n_l, t);
        const float g = __shfl_sync(0xffffffffu, g_l, t);
        if (n < begin || n >= end) continue;  // another shard's expert
        const __nv_bfloat16* we = W + (size_t)(n - begin) * d;
        const __nv_bfloat16* ve = V + (size_t)(n - begin) * d;
        uint4 wv[NV], vv[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          wv[j] = ld_vec(we + (j * 32 + lane) * 8);
          vv[j] = ld_vec(ve + (j * 32 + lane) * 8);
        }
        float zp[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          float t2 = dot2_bf16(0.f, xv[j].x, wv[j].x);
          t2 = dot2_bf16(t2, xv[j].y, wv[j].y);
          t2 = dot2_bf16(t2, xv[j].z, wv[j].z);
          zp[j] = dot2_bf16(t2, xv[j].w, wv[j].w);
        }
        float z = 0.f;
#pragma unroll
        for (int j = 0; j < NV; ++j) z += zp[j];
        z = warp_sum(z);
        const float a = g * (act == OMNIMOE_IDENTITY ? z : silu_f(z));
        const unsigned long long a2 = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          axpy2_bf16(acc[j][0], a2, vv[j].x);
          axpy2_bf16(acc[j][1], a2, vv[j].y);
          axpy2_bf16(acc[j][2], a2, vv[j].z);
          axpy2_bf16(acc[j][3], a2, vv[j].w);
        }
      }
    }
    float* yl = y + (size_t)l * d;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      float4* dst = reinterpret_cast<float4*>(yl + (j * 32 + lane) * 8);
      float4 a = make_float4(lo_f(acc[j][0]), hi_f(acc[j][0]), lo_f(acc[j][1]), hi_f(acc[j][1]));
      float4 b = make_float4(lo_f(acc[j][2]), hi_f(acc[j][2]), lo_f(acc[j][3]), hi_f(acc[j][3]));
      if (accumulate) {
        const float4 p = dst[0], q = dst[1];
        a.x += p.x; a.y += p.y; a.z += p.z; a.w += p.w;
        b.x += q.x; b.y += q.y; b.z += q.z; b.w += q.w;
      }
      dst[0] = a;
      dst[1] = b;
    }
  }
}

// ---------------------------------------------------------------------------
// expert_run_reg_kernel: run-major ECS executor with register loads (no shared
// memory staging): one warp per run (group q, token l), runs claimed 4 at a time
// in plan order; w_e, v_e loaded straight into registers for each task (L2-resident
// within the group window), x_l and the fp32 partial y_l held in registers over the
// run, one red.v4 scatter per run.  Task metadata for 32 tasks is loaded at once
// (one per lane) and broadcast by shuffle.  Same arithmetic as the TMA kernel.
template <int NV>
__global__ void __launch_bounds__(256)
    expert_run_reg_kernel(int d, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ W,
                          const __nv_bfloat16* __restrict__ V, const int32_t* __restrict__ run_off,
                          const int32_t* __restrict__ n_runs_p, const int32_t* __restrict__ m_loc_p,
                          const int32_t* __restrict__ stok, const int32_t* __restrict__ sexp,
                          const float* __restrict__ sgate, float* __restrict__ y, int act,
                          int* __restrict__ work) {
  constexpr int kChunk = 4;
  const int lane = threadIdx.x & 31;
  const int n_runs = *n_runs_p, m_loc = *m_loc_p;
  int r0 = 0;
  if (lane == 0) r0 = atomicAdd(work, kChunk);
  r0 = __shfl_sync(0xffffffffu, r0, 0);
  while (r0 < n_runs) {
    const int rend = min(r0 + kChunk, n_runs);
    const int beg0 = run_off[r0];
    const int end0 = rend < n_runs ? run_off[rend] : m_loc;
    // run starts of this chunk, lane i holds run r0 + i
    const int rs = (lane < rend - r0) ? run_off[r0 + lane] : end0;
    for (int r = r0; r < rend; ++r) {
      const int beg = __shfl_sync(0xffffffffu, rs, r - r0);
      const int end = (r + 1 < rend) ? __shfl_sync(0xffffffffu, rs, r + 1 - r0) : end0;
      const int l = stok[beg];
      uint4 xv[NV];
      unsigned long long acc[NV][4];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        xv[j] = ld_vec(x + (size_t)l * d + (j * 32 + lane) * 8);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] = 0ull;
      }
      for (int p0 = beg; p0 < end; p0 += 32) {
        const int pl = p0 + lane;
        const int e_l = pl < end ? sexp[pl] : 0;
        const float g_l = pl < end ? sgate[pl] : 0.f;
        const int cnt = min(32, end - p0);
        for (int t = 0; t < cnt; ++t) {
          const int e = __shfl_sync(0xffffffffu, e_l, t);
          const float g = __shfl_sync(0xffffffffu, g_l, t);
          const __nv_bfloat16* we = W + (size_t)e * d;
          const __nv_bfloat16* ve = V + (size_t)e * d;
          uint4 wv[NV], vv[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            wv[j] = ld_vec(we + (j * 32 + lane) * 8);
            vv[j] = ld_vec(ve + (j * 32 + lane) * 8);
          }
          float zp[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            float t2 = dot2_bf16(0.f, xv[j].x, wv[j].x);
            t2 = dot2_bf16(t2, xv[j].y, wv[j].y);
            t2 = dot2_bf16(t2, xv[j].z, wv[j].z);
            zp[j] = dot2_bf16(t2, xv[j].w, wv[j].w);
          }
          float z = 0.f;
#pragma unroll
          for (int j = 0; j < NV; ++j) z += zp[j];
          z = warp_sum(z);
          const float a = g * (act == OMNIMOE_IDENTITY ? z : silu_f(z));
          const unsigned long long a2 = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            axpy2_bf16(acc[j][0], a2, vv[j].x);
            axpy2_bf16(acc[j][1], a2, vv[j].y);
            axpy2_bf16(acc[j][2], a2, vv[j].z);
            axpy2_bf16(acc[j][3], a2, vv[j].w);
          }
        }
      }
      float* yl = y + (size_t)l * d;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * 8;
        red_add_v4(yl + c, lo_f(acc[j][0]), hi_f(acc[j][0]), lo_f(acc[j][1]), hi_f(acc[j][1]));
        red_add_v4(yl + c + 4, lo_f(acc[j][2]), hi_f(acc[j][2]), lo_f(acc[j][3]), hi_f(acc[j][3]));
      }
    }
    (void)beg0;
    if (lane == 0) r0 = atomicAdd(work, kChunk);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
  }
}

template <int NV>
omnimoe_status launch_run_reg(int d, const void* x, const void* W, const void* V, const omnimoe_plan& plan,
                              const int32_t* m_loc, float* y, int act, int* work, cudaStream_t st) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expert_run_reg_kernel<NV>, 256, 0);
  expert_run_reg_kernel<NV><<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(
      d, static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(W),
      static_cast<const __nv_bfloat16*>(V), plan.run_offsets, plan.n_runs, m_loc, plan.sorted_token,
      plan.sorted_expert, plan.sorted_gate, y, act, work);
  OMNI_CHECK_LAUNCH("expert_run_reg_kernel");
  return OMNIMOE_OK;
}

template <typename T>
omnimoe_status launch_group(int d, const void* x, const void* W, const void* V, const omnimoe_plan& plan,
                            int64_t n_loc, float* y, int act, int* work, cudaStream_t st) {
  constexpr int E = VecT<T>::E;
  const int nv = (d + 32 * E - 1) / (32 * E);
  auto X = static_cast<const T*>(x);
  auto Wp = static_cast<const T*>(W);
  auto Vp = static_cast<const T*>(V);
  const int32_t* m_loc = plan.expert_offsets + n_loc;
  // register-load run kernel for d <= 1024 (enough warps resident to hide L2 latency);
  // TMA-staged kernel above that (profiles/r1/sweep_executors.log)
  const bool reg = tuning().group_kernel >= 0 ? tuning().group_kernel == 1 : d <= 1024;
  if (sizeof(T) == 2 && d % 256 == 0 && d <= 2048 && reg) {
    switch (d / 256) {
      case 1: return launch_run_reg<1>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 2: return launch_run_reg<2>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 3: return launch_run_reg<3>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 4: return launch_run_reg<4>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 5: return launch_run_reg<5>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 6: return launch_run_reg<6>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 7: return launch_run_reg<7>(d, x, W, V, plan, m_loc, y, act, work, st);
      default: return launch_run_reg<8>(d, x, W, V, plan, m_loc, y, act, work, st);
    }
  }
  if (sizeof(T) == 2 && d % 256 == 0 && d <= 2048) {
    switch (d / 256) {
      case 1: return launch_group_tma<1, 8>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 2: return launch_group_tma<2, 6>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 3: return launch_group_tma<3, 4>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 4: return launch_group_tma<4, 4>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 5: return launch_group_tma<5, 4>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 6: return launch_group_tma<6, 3>(d, x, W, V, plan, m_loc, y, act, work, st);
      case 7: return launch_group_tma<7, 3>(d, x, W, V, plan, m_loc, y, act, work, st);
      default: return launch_group_tma<8, 3>(d, x, W, V, plan, m_loc, y, act, work, st);
    }
  }
#define OMNI_GROUP_CASE(NVC)                                                                          \
  case NVC: {                                                                                         \
    int per_sm = 1;                                                                                   \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expert_group_kernel<T, NVC>, 256, 0);      \
    expert_group_kernel<T, NVC><<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(                          \
        d, X, Wp, Vp, plan.run_offsets, plan.n_runs, m_loc, plan.sorted_token, plan.sorted_expert,    \
        plan.sorted_gate, y, act, work);                                                              \
    break;                                                                                            \
  }
  switch (nv) {
    OMNI_GROUP_CASE(1)
    OMNI_GROUP_CASE(2)
    OMNI_GROUP_CASE(4)
    OMNI_GROUP_CASE(8)
    OMNI_GROUP_CASE(16)  // fp32 at d = 2048 (all-fp32 mode at the paper's width)
    default:
      if (nv == 3) {
        expert_group_kernel<T, 4><<<num_sms() * 4, 256, 0, st>>>(d, X, Wp, Vp, plan.run_offsets, plan.n_runs, m_loc,
                                                             plan.sorted_token, plan.sorted_expert,
                                                             plan.sorted_gate, y, act, work);
        break;
      }
      if (nv <= 8) {
        expert_group_kernel<T, 8><<<num_sms() * 4, 256, 0, st>>>(d, X, Wp, Vp, plan.run_offsets, plan.n_runs, m_loc,
                                                             plan.sorted_token, plan.sorted_expert,
                                                             plan.sorted_gate, y, act, work);
        break;
      }
      set_error("expert_fwd: d too large for the grouped kernel (d <= " + std::to_string(256 * E) + ")");
      return OMNIMOE_ERR_UNSUPPORTED;
  }
#undef OMNI_GROUP_CASE
  OMNI_CHECK_LAUNCH("expert_group_kernel");
  return OMNIMOE_OK;
}

template <typename T>
omnimoe_status launch_warp(int d, const void* x, const void* W, const void* V,
                           const omnimoe_plan& plan, float* y, int act, cudaStream_t st) {
  constexpr int E = VecT<T>::E;
  const int nv = (d + 32 * E - 1) / (32 * E);
  const int grid = num_sms() * 8;
  auto X = static_cast<const T*>(x);
  auto Wp = static_cast<const T*>(W);
  auto Vp = static_cast<const T*>(V);
#define OMNI_EXPERT_CASE(NVC)                                                                       \
  case NVC:                                                                                        \
    expert_warp_kernel<T, NVC><<<grid, 256, 0, st>>>(d, X, Wp, Vp, plan.expert_offsets, plan.active, \
                                                     plan.n_active, plan.sorted_token,              \
                                                     plan.sorted_gate, y, act);                     \
    break;
  switch (nv) {
    OMNI_EXPERT_CASE(1)
    OMNI_EXPERT_CASE(2)
    OMNI_EXPERT_CASE(3)
    OMNI_EXPERT_CASE(4)
    OMNI_EXPERT_CASE(6)
    OMNI_EXPERT_CASE(8)
    OMNI_EXPERT_CASE(16)
    default:
      if (nv <= 16) {
        expert_warp_kernel<T, 16><<<grid, 256, 0, st>>>(d, X, Wp, Vp, plan.expert_offsets, plan.active,
                                                       plan.n_active, plan.sorted_token,
                                                       plan.sorted_gate, y, act);
        break;
      }
      set_error("expert_fwd: d too large for the register-resident expert kernel (d <= " +
                std::to_string(512 * E) + ")");
      return OMNIMOE_ERR_UNSUPPORTED;
  }
#undef OMNI_EXPERT_CASE
  OMNI_CHECK_LAUNCH("expert_warp_kernel");
  return OMNIMOE_OK;
}


// ---------------------------------------------------------------------------
// SLICED executor (dims.v_layout == OMNIMOE_V_SLICED).
//
// Per task the method needs one d-row of W (for z) and one d-row of V (for the
// axpy); with random routing the only reuse is across the eta = M/|E_active|
// tasks of an expert, so those rows cross L2 -> SM once per task whatever the
// loop order, and every re-read that misses L2 costs HBM.  The executor splits
// Eq.Grouped into two passes so that each keeps its working set in L2:
//
//  expert_dot_kernel (pass Z): the plan's runs (group q, token l) in plan order,
//    x_l in registers, w_e streamed (the group's W rows stay L2-resident: D_expert
//    once from HBM), a_t = g * sigma(x_l . w_e) written to task_pair[t][1].
//  expert_vslice_kernel (pass V): slice-major.  For slice s (32 columns) every
//    token l gathers the 64-byte slice of v_e of each of its tasks (token order,
//    plan->token_offsets), accumulates a_t * v_e[s] in registers and writes its
//    y_routed slice once.  The whole slice of V (64 N bytes, 67 MB at N = 2^20) is
//    L2-resident while all tokens use it, so V is read from HBM once, and no
//    atomics touch y_routed.
template <int NV>
__global__ void __launch_bounds__(256)
    expert_dot_kernel(int d, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ W,
                      const int32_t* __restrict__ run_off, const int32_t* __restrict__ n_runs_p,
                      const int32_t* __restrict__ m_loc_p, const int32_t* __restrict__ stok,
                      const int32_t* __restrict__ sexp, const float* __restrict__ sgate,
                      const int32_t* __restrict__ stask, int32_t* __restrict__ task_pair, int act,
                      int* __restrict__ work) {
  constexpr int kChunk = 4;
  const int lane = threadIdx.x & 31;
  const int n_runs = *n_runs_p, m_loc = *m_loc_p;
  int r0 = 0;
  if (lane == 0) r0 = atomicAdd(work, kChunk);
  r0 = __shfl_sync(0xffffffffu, r0, 0);
  while (r0 < n_runs) {
    const int rend = min(r0 + kChunk, n_runs);
    const int end0 = rend < n_runs ? run_off[rend] : m_loc;
    const int rs = (lane < rend - r0) ? run_off[r0 + lane] : end0;  // lane i: start of run r0 + i
    for (int r = r0; r < rend; ++r) {
      const int beg = __shfl_sync(0xffffffffu, rs, r - r0);
      const int end = (r + 1 < rend) ? __shfl_sync(0xffffffffu, rs, r + 1 - r0) : end0;
      const int l = stok[beg];
      uint4 xv[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int c = (j * 32 + lane) * 8;
        xv[j] = c < d ? ld_vec(x + (size_t)l * d + c) : make_uint4(0, 0, 0, 0);
      }
      for (int p0 = beg; p0 < end; p0 += 32) {
        const int pl = p0 + lane;
        const int e_l = pl < end ? sexp[pl] : 0;
        const float g_l = pl < end ? sgate[pl] : 0.f;
        const int t_l = pl < end ? stask[pl] : 0;
        const int cnt = min(32, end - p0);
        float my_a = 0.f;
        for (int t = 0; t < cnt; t += 2) {  // two tasks in flight per warp
          const int t1 = min(t + 1, cnt - 1);
          const int e0 = __shfl_sync(0xffffffffu, e_l, t), e1 = __shfl_sync(0xffffffffu, e_l, t1);
          const float g0 = __shfl_sync(0xffffffffu, g_l, t), g1 = __shfl_sync(0xffffffffu, g_l, t1);
          const __nv_bfloat16* w0 = W + (size_t)e0 * d;
          const __nv_bfloat16* w1 = W + (size_t)e1 * d;
          uint4 a[NV], b[NV];
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            const int c = (j * 32 + lane) * 8;
            a[j] = c < d ? ld_vec(w0 + c) : make_uint4(0, 0, 0, 0);
            b[j] = c < d ? ld_vec(w1 + c) : make_uint4(0, 0, 0, 0);
          }
          float z0 = 0.f, z1 = 0.f;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            float u = dot2_bf16(0.f, xv[j].x, a[j].x);
            u = dot2_bf16(u, xv[j].y, a[j].y);
            u = dot2_bf16(u, xv[j].z, a[j].z);
            z0 += dot2_bf16(u, xv[j].w, a[j].w);
            float v = dot2_bf16(0.f, xv[j].x, b[j].x);
            v = dot2_bf16(v, xv[j].y, b[j].y);
            v = dot2_bf16(v, xv[j].z, b[j].z);
            z1 += dot2_bf16(v, xv[j].w, b[j].w);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            z0 += __shfl_xor_sync(0xffffffffu, z0, o);
            z1 += __shfl_xor_sync(0xffffffffu, z1, o);
          }
          const float a0 = g0 * (act == OMNIMOE_IDENTITY ? z0 : silu_f(z0));
          const float a1 = g1 * (act == OMNIMOE_IDENTITY ? z1 : silu_f(z1));
          if (lane == t) my_a = a0;
          if (lane == t + 1) my_a = a1;
        }
        if (lane < cnt) task_pair[2 * (size_t)t_l + 1] = __float_as_int(my_a);
      }
    }
    if (lane == 0) r0 = atomicAdd(work, kChunk);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
  }
}

__device__ __forceinline__ int2 ld_pair(const int32_t* p, uint64_t pol) {
  int2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return r;
}

// 32-byte load (LDG.256, sm_100): 16 bf16 of a 128-byte V slice piece
struct U8 {
  uint32_t w[8];
};
__device__ __forceinline__ U8 ld256(const void* p) {
  U8 r;
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                 "=r"(r.w[7])
               : "l"(p));
  return r;
}

// pass V: one warp per (slice, token) item over the SLICED layout [d/64][n][64] (one
// 128-byte piece per expert and slice); lane = (task sub-slot g8 = lane / 4, 32-byte
// quarter c4 = lane % 4 of the piece): 8 tasks per 256-bit load instruction, 16 bf16
// columns per lane.  The (expert, a) pairs of the next window -- possibly of the next
// item, which is claimed one item ahead -- are loaded while the current one is
// processed.  Items (slice, token) are claimed in order from one counter so that the
// warps in flight stay within ~one slice (a static round-robin lets warps drift over
// many slices: C3a pass V 3.45 -> 13.6 ms in round 1).
// BF16A: the task's coefficient a_t is rounded to bf16 and multiplied with the bf16 slice
// elements by fma.rn.f32.bf16 (FHFMA, one instruction per element, fp32 accumulation),
// instead of unpacking the pieces to fp32 for FFMA2 (three instructions per two elements;
// the unpack was 30 % of the kernel's instructions).  Reading Q21: the
// forward's activations a_t = g_t SiLU(z_t) enter the scatter-accumulate in bf16, as the
// paper's bf16 kernels hold them; the backward's dz keeps fp32 (BF16A = false).
template <int MINB, int W, bool BF16A>
__global__ void __launch_bounds__(256, MINB)
    expert_vslice_kernel(int d, int64_t L, int64_t n_loc, const int32_t* __restrict__ seg, int seg_stride,
                         int band, int64_t n_tok, const int32_t* __restrict__ task_pair,
                         const __nv_bfloat16* __restrict__ Vs, float* __restrict__ y, int accumulate,
                         int* __restrict__ work) {
  constexpr int WT = 8 * W;    // tasks per window: W rounds of 8 tasks, one 32-byte load per lane each
  constexpr int NP = (WT + 31) / 32;  // (expert, a) pairs per lane and window
  const int lane = threadIdx.x & 31, c4 = lane & 3, g8 = lane >> 2;
  const int S = d / 64;
  const int64_t n_items = (int64_t)S * L;
  const uint64_t pol = policy_evict_first();
  auto claim = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(work, 1);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  auto range = [&](int64_t item, int& beg, int& end) {
    beg = end = 0;
    if (item < n_items) {
      const int64_t l = item % L;
      if (l < n_tok) {
        beg = seg[l * seg_stride + band];
        end = seg[l * seg_stride + band + 1];
      }
    }
  };
  auto fetch = [&](int p0, int end, int2 (&pp)[NP]) {
#pragma unroll
    for (int k = 0; k < NP; ++k)
      pp[k] = (32 * k + lane < WT && p0 + 32 * k + lane < end)
                  ? ld_pair(task_pair + 2 * (size_t)(p0 + 32 * k + lane), pol)
                  : make_int2(-1, 0);
  };
  // the output quarter this lane adds to (band > 0 or accumulate) is copied into shared
  // memory by cp.async when the item starts and read when it ends: no dependent round
  // trip at the end of the item and no registers held across it
  __shared__ __align__(16) float ysm[8][4][16];
  __shared__ __align__(16) float rsm[8][8 * 68];
  float* my_y = ysm[threadIdx.x >> 5][c4];
  int64_t it = claim();
  int beg, end;
  range(it, beg, end);
  int2 np_[NP];
  fetch(beg, end, np_);
  while (it < n_items) {
    const int64_t nxt = claim();
    int nbeg, nend;
    range(nxt, nbeg, nend);
    const int s = (int)(it / L);
    const int64_t l = it - (int64_t)s * L;
    float* yq = y + (size_t)l * d + s * 64 + c4 * 16;
    if (accumulate && g8 == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(my_y + 4 * q)), "l"(yq + 4 * q)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const __nv_bfloat16* vs = Vs + (size_t)s * n_loc * 64 + c4 * 16;
    unsigned long long acc[8];
    float fa[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0ull;
#pragma unroll
    for (int i = 0; i < 16; ++i) fa[i] = 0.f;
    for (int p0 = beg; p0 < end; p0 += WT) {
      int2 cp[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) cp[k] = np_[k];
      if (p0 + WT < end) fetch(p0 + WT, end, np_);
      else fetch(nbeg, nend, np_);  // the next item's first tasks
      const int n_r = min(W, (end - p0 + 7) >> 3);  // rounds of 8 tasks holding work
      U8 v[W];
      float a[W];
#pragma unroll
      for (int r = 0; r < W; ++r) {
        const int src = (r & 3) * 8 + g8;
        const int e = __shfl_sync(0xffffffffu, cp[r >> 2].x, src);
        a[r] = __int_as_float(__shfl_sync(0xffffffffu, cp[r >> 2].y, src));
        if (e < 0) a[r] = 0.f;
        if (r < n_r && e >= 0) {
          v[r] = ld256(vs + (size_t)e * 64);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[r].w[i] = 0u;
        }
      }
#pragma unroll
      for (int r = 0; r < W; ++r) {
        if (BF16A) {
          const unsigned short ab = __bfloat16_as_ushort(__float2bfloat16_rn(a[r]));
#pragma unroll
          for (int i = 0; i < 8; ++i) fma_bf16_pair(fa[2 * i], fa[2 * i + 1], ab, v[r].w[i]);
        } else {
          const unsigned long long a2 = ((unsigned long long)__float_as_uint(a[r]) << 32) | __float_as_uint(a[r]);
#pragma unroll
          for (int i = 0; i < 8; ++i) axpy2_bf16(acc[i], a2, v[r].w[i]);
        }
      }
    }
    if (beg == end) fetch(nbeg, nend, np_);
    // the 8 task groups' partial sums of the slice's 64 columns go through shared memory
    // (rows padded to 68 floats): lane j then adds columns 2j, 2j+1 over the 8 rows and
    // writes them with one coalesced 256-byte store per warp -- instead of 48 shuffles
    // + 48 adds per lane and 4 writing lanes
    float* red = rsm[threadIdx.x >> 5];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 u;
      if (BF16A) {
        u = make_float4(fa[4 * q], fa[4 * q + 1], fa[4 * q + 2], fa[4 * q + 3]);
      } else {
        u = make_float4(lo_f(acc[2 * q]), hi_f(acc[2 * q]), lo_f(acc[2 * q + 1]), hi_f(acc[2 * q + 1]));
      }
      *reinterpret_cast<float4*>(red + g8 * 68 + c4 * 16 + 4 * q) = u;
    }
    if (accumulate && g8 == 0) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    float2 sum = *reinterpret_cast<const float2*>(red + 2 * lane);
#pragma unroll
    for (int g = 1; g < 8; ++g) {
      const float2 t = *reinterpret_cast<const float2*>(red + g * 68 + 2 * lane);
      sum.x += t.x;
      sum.y += t.y;
    }
    if (accumulate) {
      const float2 p = reinterpret_cast<const float2*>(ysm[threadIdx.x >> 5])[lane];
      sum.x += p.x;
      sum.y += p.y;
    }
    *reinterpret_cast<float2*>(y + (size_t)l * d + s * 64 + 2 * lane) = sum;
    __syncwarp();  // red and the prefetched output slice are reused by the next item
    it = nxt;
    beg = nbeg;
    end = nend;
  }
}

// pass V for few tasks per token (h*K <= 64): one warp per (slice, 8 consecutive
// tokens), lane group g8 = lane / 4 owns one token, 4 of its tasks per step (one
// 32-byte quarter of each 128-byte piece per lane); no cross-lane reduction.
__global__ void __launch_bounds__(256)
    expert_vslice_group_kernel(int d, int64_t L, int64_t n_loc, const int32_t* __restrict__ seg, int seg_stride,
                               int band, int64_t n_tok, const int32_t* __restrict__ task_pair,
                               const __nv_bfloat16* __restrict__ Vs, float* __restrict__ y, int accumulate,
                               int* __restrict__ work) {
  constexpr int T = 4;
  const int lane = threadIdx.x & 31, c4 = lane & 3, g8 = lane >> 2;
  const int S = d / 64;
  const int64_t n_tc = (L + 7) / 8;
  const int64_t n_items = (int64_t)S * n_tc;
  const uint64_t pol = policy_evict_first();
  auto claim = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(work, 1);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  for (int64_t it = claim(); it < n_items; it = claim()) {
    const int s = (int)(it / n_tc);
    const int64_t l = (it - (int64_t)s * n_tc) * 8 + g8;
    int beg = 0, n = 0;
    if (l < L && l < n_tok) {
      beg = seg[l * seg_stride + band];
      n = seg[l * seg_stride + band + 1] - beg;
    }
    const __nv_bfloat16* vs = Vs + (size_t)s * n_loc * 64 + c4 * 16;
    const int nmax = __reduce_max_sync(0xffffffffu, n);
    unsigned long long acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0ull;
    int2 nx[T];  // the (expert, a) pairs of the next T tasks, loaded one step ahead
#pragma unroll
    for (int t = 0; t < T; ++t) nx[t] = t < n ? ld_pair(task_pair + 2 * (size_t)(beg + t), pol) : make_int2(-1, 0);
    for (int q = 0; q < nmax; q += T) {
      int2 pr[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        pr[t] = nx[t];
        nx[t] = q + T + t < n ? ld_pair(task_pair + 2 * (size_t)(beg + q + T + t), pol) : make_int2(-1, 0);
      }
      U8 v[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        if (pr[t].x >= 0) {
          v[t] = ld256(vs + (size_t)pr[t].x * 64);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[t].w[i] = 0u;
        }
      }
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const float a = pr[t].x >= 0 ? __int_as_float(pr[t].y) : 0.f;
        const unsigned long long a2 = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
#pragma unroll
        for (int i = 0; i < 8; ++i) axpy2_bf16(acc[i], a2, v[t].w[i]);
      }
    }
    if (l < L) {
      float4* dst = reinterpret_cast<float4*>(y + (size_t)l * d + s * 64 + c4 * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 u = make_float4(lo_f(acc[2 * q]), hi_f(acc[2 * q]), lo_f(acc[2 * q + 1]), hi_f(acc[2 * q + 1]));
        if (accumulate) {
          const float4 p = dst[q];
          u.x += p.x; u.y += p.y; u.z += p.z; u.w += p.w;
        }
        dst[q] = u;
      }
    }
  }
}

// V [n][d] -> V_sliced [d/64][n][64] (16-byte moves; bit-exact)
__global__ void pack_v_kernel(const uint4* __restrict__ V, uint4* __restrict__ Vs, int64_t n, int d) {
  const int64_t per_row = d / 8, total = n * per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / per_row;
    const int q = (int)(i - row * per_row);
    Vs[((size_t)(q >> 3) * n + row) * 8 + (q & 7)] = V[i];
  }
}


// pass Z on an expert-major plan (B = 1): one warp per active
// expert holds w_e in registers (W streamed from HBM once, in ascending expert
// order) and walks the expert's tasks: x_l gathered from L2 (x is the only
// reused operand: 2dL bytes), a_t = g * sigma(x_l . w_e) -> task_pair[t][1].  Two
// tasks' x rows are in flight per warp.
template <int NV, int MINB, int T>
__global__ void __launch_bounds__(256, MINB)
    expert_zdot_kernel(int d, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ W,
                       const int32_t* __restrict__ offsets, const int32_t* __restrict__ active,
                       const int32_t* __restrict__ n_active, const int32_t* __restrict__ stok,
                       const float* __restrict__ sgate, const int32_t* __restrict__ stask,
                       int32_t* __restrict__ task_pair, int act, int* __restrict__ work, int w_hint, int x_hint) {
  const int lane = threadIdx.x & 31;
  const int na = *n_active;
  const uint64_t pol = w_hint ? policy_evict_first() : policy_evict_normal();
  const uint64_t xpol = x_hint ? policy_evict_last() : policy_evict_normal();
  int tau = 0;
  if (lane == 0) tau = atomicAdd(work, 1);
  tau = __shfl_sync(0xffffffffu, tau, 0);
  while (tau < na) {
    const int e = active[tau];
    const int beg = offsets[e], end = offsets[e + 1];
    uint4 wv[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * 8;
      wv[j] = c < d ? ld_vec_hint(W + (size_t)e * d + c, pol) : make_uint4(0, 0, 0, 0);
    }
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(work, 1);  // claim the next expert early
    for (int p0 = beg; p0 < end; p0 += 32) {
      const int pl = p0 + lane;
      const int l_l = pl < end ? stok[pl] : 0;
      const float g_l = pl < end ? sgate[pl] : 0.f;
      const int t_l = pl < end ? stask[pl] : 0;
      const int cnt = min(32, end - p0);
      float my_a = 0.f;
      for (int t = 0; t < cnt; t += T) {  // T tasks' x rows in flight per warp
        int lt[T];
        uint4 xr[T][NV];
#pragma unroll
        for (int u = 0; u < T; ++u) {
          lt[u] = __shfl_sync(0xffffffffu, l_l, min(t + u, cnt - 1));
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            const int c = (j * 32 + lane) * 8;
            xr[u][j] = c < d ? ld_vec_hint(x + (size_t)lt[u] * d + c, xpol) : make_uint4(0, 0, 0, 0);
          }
        }
        float z[T];
#pragma unroll
        for (int u = 0; u < T; ++u) {
          z[u] = 0.f;
#pragma unroll
          for (int j = 0; j < NV; ++j) {
            float q = dot2_bf16(0.f, wv[j].x, xr[u][j].x);
            q = dot2_bf16(q, wv[j].y, xr[u][j].y);
            q = dot2_bf16(q, wv[j].z, xr[u][j].z);
            z[u] += dot2_bf16(q, wv[j].w, xr[u][j].w);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < T; ++u) z[u] += __shfl_xor_sync(0xffffffffu, z[u], o);
#pragma unroll
        for (int u = 0; u < T; ++u) {
          const float g = __shfl_sync(0xffffffffu, g_l, min(t + u, cnt - 1));
          const float a = g * (act == OMNIMOE_IDENTITY ? z[u] : silu_f(z[u]));
          if (lane == t + u) my_a = a;
        }
      }
      if (lane < cnt) task_pair[2 * (size_t)t_l + 1] = __float_as_int(my_a);
    }
    tau = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

// pass Z with 32-byte loads (LDG.256): the same arithmetic and order of work as
// expert_zdot_kernel, half the load instructions per row (d % 512 == 0)
__device__ __forceinline__ U8 ld256_hint(const void* p, uint64_t pol) {
  U8 r;
  asm volatile("ld.global.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
                 "=r"(r.w[7])
               : "l"(p), "l"(pol));
  return r;
}

template <int NV8, int MINB, int T>
__global__ void __launch_bounds__(256, MINB)
    expert_zdot256_kernel(int d, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ W,
                          const int32_t* __restrict__ offsets, const int32_t* __restrict__ active,
                          const int32_t* __restrict__ n_active, const int32_t* __restrict__ stok,
                          const float* __restrict__ sgate, const int32_t* __restrict__ stask,
                          int32_t* __restrict__ task_pair, int act, int* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  const int na = *n_active;
  const uint64_t pol = policy_evict_first(), xpol = policy_evict_normal();
  int tau = 0;
  if (lane == 0) tau = atomicAdd(work, 1);
  tau = __shfl_sync(0xffffffffu, tau, 0);
  while (tau < na) {
    const int e = active[tau];
    const int beg = offsets[e], end = offsets[e + 1];
    U8 wv[NV8];
#pragma unroll
    for (int j = 0; j < NV8; ++j) wv[j] = ld256_hint(W + (size_t)e * d + (j * 32 + lane) * 16, pol);
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(work, 1);  // claim the next expert early
    for (int p0 = beg; p0 < end; p0 += 32) {
      const int pl = p0 + lane;
      const int l_l = pl < end ? stok[pl] : 0;
      const float g_l = pl < end ? sgate[pl] : 0.f;
      const int t_l = pl < end ? stask[pl] : 0;
      const int cnt = min(32, end - p0);
      float my_a = 0.f;
      for (int t = 0; t < cnt; t += T) {
        U8 xr[T][NV8];
#pragma unroll
        for (int u = 0; u < T; ++u) {
          const int lt = __shfl_sync(0xffffffffu, l_l, min(t + u, cnt - 1));
#pragma unroll
          for (int j = 0; j < NV8; ++j) xr[u][j] = ld256_hint(x + (size_t)lt * d + (j * 32 + lane) * 16, xpol);
        }
        float z[T];
#pragma unroll
        for (int u = 0; u < T; ++u) {
          z[u] = 0.f;
#pragma unroll
          for (int j = 0; j < NV8; ++j) {
            float q = 0.f, q2 = 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              q = dot2_bf16(q, wv[j].w[i], xr[u][j].w[i]);
              q2 = dot2_bf16(q2, wv[j].w[4 + i], xr[u][j].w[4 + i]);
            }
            z[u] += q + q2;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < T; ++u) z[u] += __shfl_xor_sync(0xffffffffu, z[u], o);
#pragma unroll
        for (int u = 0; u < T; ++u) {
          const float g = __shfl_sync(0xffffffffu, g_l, min(t + u, cnt - 1));
          const float a = g * (act == OMNIMOE_IDENTITY ? z[u] : silu_f(z[u]));
          if (lane == t + u) my_a = a;
        }
      }
      if (lane < cnt) task_pair[2 * (size_t)t_l + 1] = __float_as_int(my_a);
    }
    tau = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

template <int NV>
omnimoe_status launch_zdot(int d, const void* x, const void* W, const omnimoe_plan& plan, int act, int* work,
                           cudaStream_t st) {
  auto go = [&](auto kern) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
    kern<<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(
        d, static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(W), plan.expert_offsets,
        plan.active, plan.n_active, plan.sorted_token, plan.sorted_gate, plan.sorted_task, plan.task_pair, act, work,
        tuning().w_hint, tuning().x_hint);
  };
  // 80 registers (3 CTAs per SM) with two x rows in flight per warp: pass Z 3.27 -> 2.25 ms at
  // C3a against 64 registers / 4 CTAs (profiles/r2/occupancy/); 2 CTAs or 4 rows in flight: no gain
  go(expert_zdot_kernel<NV, 3, 2>);
  OMNI_CHECK_LAUNCH("expert_zdot_kernel");
  return OMNIMOE_OK;
}

template <int NV>
omnimoe_status launch_dot(int d, const void* x, const void* W, const omnimoe_plan& plan, const int32_t* m_loc,
                          int act, int* work, cudaStream_t st) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expert_dot_kernel<NV>, 256, 0);
  expert_dot_kernel<NV><<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(
      d, static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(W), plan.run_offsets, plan.n_runs,
      m_loc, plan.sorted_token, plan.sorted_expert, plan.sorted_gate, plan.sorted_task, plan.task_pair, act, work);
  OMNI_CHECK_LAUNCH("expert_dot_kernel");
  return OMNIMOE_OK;
}


// ---------------------------------------------------------------------------
// N2: backward of the routed branch for a fixed routing decision,
// on the expert-major plan (B = 1): a PAIR of warps per active expert, warp h of the
// pair owning columns [h d/2, (h+1) d/2): w_e and v_e halves in registers; per task
// the x_l and dy_l halves are gathered, the partial dots z = x_l . w_e and
// q = dy_l . v_e are exchanged through shared memory (double-buffered, one named
// barrier per task), then dV_e += g s(z) dy_l and dW_e += dz x_l accumulate in
// registers (dz = g q s'(z)), and the expert's dW, dV rows are written once --
// no atomics.  Per task: dgate = s(z) q (task order) and dz into task_pair.y for the
// token-stationary dx pass (expert_vslice_kernel over the sliced W).
template <int NVH, int G>
__global__ void __launch_bounds__(256)
    expert_bwd_kernel(int d, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ W,
                      const __nv_bfloat16* __restrict__ V, const __nv_bfloat16* __restrict__ dy,
                      const int32_t* __restrict__ offsets, const int32_t* __restrict__ active,
                      const int32_t* __restrict__ n_active, const int32_t* __restrict__ stok,
                      const float* __restrict__ sgate, const int32_t* __restrict__ stask,
                      int32_t* __restrict__ task_pair, float* __restrict__ dgate, float* __restrict__ dW_act,
                      float* __restrict__ dV_act, int act) {
  constexpr int kGroups = 8 / G;  // expert groups (of G warps) per CTA
  __shared__ float xch[kGroups][2][G][2];  // [group][parity][part][z, q]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, pair = warp / G, h = warp % G;
  const int half = d / G, c0 = h * half;  // this warp's column part
  const int na = *n_active;
  const int np = gridDim.x * kGroups;
  int parity = 0;
  for (int tau = blockIdx.x * kGroups + pair; tau < na; tau += np) {
    const int e = active[tau];
    const int beg = offsets[e], end = offsets[e + 1];
    uint4 wv[NVH], vv[NVH];
    unsigned long long aw[NVH][4], av[NVH][4];
#pragma unroll
    for (int j = 0; j < NVH; ++j) {
      const int c = (j * 32 + lane) * 8;
      wv[j] = c < half ? ld_vec(W + (size_t)e * d + c0 + c) : make_uint4(0, 0, 0, 0);
      vv[j] = c < half ? ld_vec(V + (size_t)e * d + c0 + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int i = 0; i < 4; ++i) aw[j][i] = av[j][i] = 0ull;
    }
    // the next task's x and dy parts (and gate, task index) are loaded one task ahead
    uint4 nxh[NVH], ndh[NVH];
    float ng = 0.f;
    int nt = 0;
    auto fetch = [&](int p) {
      if (p >= end) return;
      const int l = stok[p];
      ng = sgate[p];
      nt = stask[p];
#pragma unroll
      for (int j = 0; j < NVH; ++j) {
        const int c = (j * 32 + lane) * 8;
        nxh[j] = c < half ? ld_vec(x + (size_t)l * d + c0 + c) : make_uint4(0, 0, 0, 0);
        ndh[j] = c < half ? ld_vec(dy + (size_t)l * d + c0 + c) : make_uint4(0, 0, 0, 0);
      }
    };
    fetch(beg);
    for (int p = beg; p < end; ++p) {
      const float g = ng;
      const int tcur = nt;
      uint4 xh[NVH], dh[NVH];
#pragma unroll
      for (int j = 0; j < NVH; ++j) {
        xh[j] = nxh[j];
        dh[j] = ndh[j];
      }
      fetch(p + 1);
      float zp = 0.f, qp = 0.f;
#pragma unroll
      for (int j = 0; j < NVH; ++j) {
        float u = dot2_bf16(0.f, xh[j].x, wv[j].x);
        u = dot2_bf16(u, xh[j].y, wv[j].y);
        u = dot2_bf16(u, xh[j].z, wv[j].z);
        zp += dot2_bf16(u, xh[j].w, wv[j].w);
        float v = dot2_bf16(0.f, dh[j].x, vv[j].x);
        v = dot2_bf16(v, dh[j].y, vv[j].y);
        v = dot2_bf16(v, dh[j].z, vv[j].z);
        qp += dot2_bf16(v, dh[j].w, vv[j].w);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        zp += __shfl_xor_sync(0xffffffffu, zp, o);
        qp += __shfl_xor_sync(0xffffffffu, qp, o);
      }
      if (lane == 0) {
        xch[pair][parity][h][0] = zp;
        xch[pair][parity][h][1] = qp;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(32 * G) : "memory");
      float z = 0.f, q = 0.f;  // the same summation order in every warp of the group
#pragma unroll
      for (int u = 0; u < G; ++u) {
        z += xch[pair][parity][u][0];
        q += xch[pair][parity][u][1];
      }
      parity ^= 1;
      const float lg = 1.0f / (1.0f + __expf(-z));
      const float sz = act == OMNIMOE_IDENTITY ? z : z * lg;
      const float sp = act == OMNIMOE_IDENTITY ? 1.0f : lg * (1.0f + z * (1.0f - lg));
      const float a = g * sz, dz = g * q * sp;
      if (h == 0 && lane == 0) {
        const int t = tcur;
        dgate[t] = sz * q;
        task_pair[2 * (size_t)t + 1] = __float_as_int(dz);
      }
      const unsigned long long a2 = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
      const unsigned long long z2 = ((unsigned long long)__float_as_uint(dz) << 32) | __float_as_uint(dz);
#pragma unroll
      for (int j = 0; j < NVH; ++j) {
        axpy2_bf16(av[j][0], a2, dh[j].x);
        axpy2_bf16(av[j][1], a2, dh[j].y);
        axpy2_bf16(av[j][2], a2, dh[j].z);
        axpy2_bf16(av[j][3], a2, dh[j].w);
        axpy2_bf16(aw[j][0], z2, xh[j].x);
        axpy2_bf16(aw[j][1], z2, xh[j].y);
        axpy2_bf16(aw[j][2], z2, xh[j].z);
        axpy2_bf16(aw[j][3], z2, xh[j].w);
      }
    }
#pragma unroll
    for (int j = 0; j < NVH; ++j) {
      const int c = (j * 32 + lane) * 8;
      if (c < half) {
        float4* dw = reinterpret_cast<float4*>(dW_act + (size_t)tau * d + c0 + c);
        float4* dv = reinterpret_cast<float4*>(dV_act + (size_t)tau * d + c0 + c);
        dw[0] = make_float4(lo_f(aw[j][0]), hi_f(aw[j][0]), lo_f(aw[j][1]), hi_f(aw[j][1]));
        dw[1] = make_float4(lo_f(aw[j][2]), hi_f(aw[j][2]), lo_f(aw[j][3]), hi_f(aw[j][3]));
        dv[0] = make_float4(lo_f(av[j][0]), hi_f(av[j][0]), lo_f(av[j][1]), hi_f(av[j][1]));
        dv[1] = make_float4(lo_f(av[j][2]), hi_f(av[j][2]), lo_f(av[j][3]), hi_f(av[j][3]));
      }
    }
  }
}

}  // namespace

size_t expert_ws_bytes(const omnimoe_dims&, int64_t) { return 256; }  // work counters

// N2 workspace: counters + z, q, dz, g s per task (upper bound L h K tasks) + the dx pass's
int64_t bwd_ws_tasks(const omnimoe_dims& d, int64_t L) { return std::max<int64_t>(L * d.n_heads * d.top_k, 1); }
size_t expert_bwd_ws_bytes(const omnimoe_dims& d, int64_t L) {
  return 256 + 16 * (size_t)bwd_ws_tasks(d, L) + expert_ws_bytes(d, L);
}

omnimoe_status expert_token_run(const omnimoe_dims& dm, int64_t L, const void* x, const void* W, const void* V,
                                const int32_t* idx, const float* gate, int64_t begin, int64_t end, float* y,
                                int accumulate, cudaStream_t st) {
  if (dm.dtype != OMNIMOE_BF16 || dm.d % 256 != 0 || dm.d > 2048) {
    set_error("token-centric executor: bf16 with d a multiple of 256, d <= 2048");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (L == 0) return OMNIMOE_OK;
  const int hk = (int)(dm.n_heads * dm.top_k);
  const int grid = (int)std::min<int64_t>((L + 7) / 8, num_sms() * 16);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto Wp = static_cast<const __nv_bfloat16*>(W);
  auto Vp = static_cast<const __nv_bfloat16*>(V);
  switch (dm.d / 256) {
#define OMNI_TOK_CASE(NVC)                                                                                       \
  case NVC:                                                                                                      \
    expert_token_kernel<NVC><<<grid, 256, 0, st>>>((int)dm.d, L, hk, X, Wp, Vp, idx, gate, begin, end, y,         \
                                                   accumulate, dm.act);                                          \
    break;
    OMNI_TOK_CASE(1)
    OMNI_TOK_CASE(2)
    OMNI_TOK_CASE(3)
    OMNI_TOK_CASE(4)
    OMNI_TOK_CASE(5)
    OMNI_TOK_CASE(6)
    OMNI_TOK_CASE(7)
    OMNI_TOK_CASE(8)
#undef OMNI_TOK_CASE
  }
  OMNI_CHECK_LAUNCH("expert_token_kernel");
  return OMNIMOE_OK;
}

int64_t resolve_group_size(const omnimoe_dims& d) {
  if (d.group_size > 0) return d.group_size;
  if (d.dtype != OMNIMOE_BF16) return 1;  // fp32 correctness mode: expert-major
  if (d.v_layout == OMNIMOE_V_SLICED) return 1;  // SLICED pass Z walks an expert-major plan
  // eight grid rows of experts per group, capped so one group's W/V rows (4d bytes
  // per expert) stay within 64 MB of L2 (tools/sweep_group.py)
  const int64_t cap = std::max<int64_t>(1, (64ll << 20) / (4 * d.d));
  return std::max<int64_t>(2, std::min<int64_t>(8 * d.n_cols, cap));
}

double expected_eta(const omnimoe_dims& d, int64_t L) {
  const double N = (double)(d.n_rows * d.n_cols), M = (double)L * d.n_heads * d.top_k;
  const double active = N * -expm1(-M / N);  // N (1 - (1 - 1/N)^M), N large
  return active > 0 ? M / active : 0.0;
}

bool layer_uses_token_executor(const omnimoe_dims& d, int64_t L) {
  if (d.expert_kernel == OMNIMOE_EXPERT_TOKEN) return true;
  // measured (profiles/r1/README.md, C3b / C5s at eta ~ 1.1): with no expert shared by two
  // tasks, scheduling and two passes cost more than they save; full-row gathers win
  return d.expert_kernel == OMNIMOE_EXPERT_AUTO && d.v_layout == OMNIMOE_V_ROWS && d.dtype == OMNIMOE_BF16 &&
         d.d % 256 == 0 && d.d <= 2048 && expected_eta(d, L) < tuning().token_eta_x100 / 100.0;
}

// pass V geometry: pass V sweeps the 64-column slices of V one band of
// experts at a time (one launch per band, item order (slice, token) inside it); the
// band's part of a slice (128 bytes per expert) is kept within dims.v_band_bytes (68 MB
// of the 126 MB L2) so that it stays resident while every token uses it.  More bands
// than that measured slower (C3a: 1 band 3.45 ms, 2 bands 3.50, 4 bands 5.16; C5: 4
// bands beat 8 -- profiles/r2/bands/): every band multiplies the (slice, token) items
// and their fixed costs, and bands > 0 re-read the output rows.
int64_t resolve_v_bands(const omnimoe_dims& d, int64_t n_loc, int64_t n_tok) {
  (void)n_tok;
  if (n_loc < 1) return 1;
  const int64_t budget = d.v_band_bytes > 0 ? d.v_band_bytes : (68ll << 20);
  const int64_t by_l2 = std::max<int64_t>(1, std::min<int64_t>(30, (128 * n_loc + budget - 1) / budget));
  if (d.v_band_bytes > 0) return by_l2;
  // but at least ~128 tasks per (token, band) item: the item's fixed costs (claim, segment
  // bounds, first pairs, reduction, output write) outweigh the L2 misses of a chunk above
  // the budget (C5: 4 bands of 134 MB 16.3 ms, 8 bands of 67 MB 19.0 ms; C3a: 2 bands of
  // 67 MB 2.82 ms, 1 band of 134 MB 3.16 ms -- profiles/r2/slices128/)
  const double N = (double)(d.n_rows * d.n_cols);
  const double tasks_per_token = (double)(d.n_heads * d.top_k) * std::min(1.0, (double)n_loc / N);
  return std::min<int64_t>(by_l2, std::max<int64_t>(1, (int64_t)(tasks_per_token / 128.0)));
}

int64_t resolve_token_blocks(const omnimoe_dims& d, int64_t L) {
  if (resolve_group_size(d) == 1) return 1;
  (void)L;
  // measured (profiles/r1/sweep_*.log): blocking the batch does not pay at C3a --
  // the W/V stream evicts y_routed between a token's runs whatever the block size
  return d.token_blocks > 0 ? d.token_blocks : 1;
}

omnimoe_status expert_sliced_run(const omnimoe_dims& dm, int64_t L, const void* x, const void* W, const void* Vs,
                                 const omnimoe_plan& plan, float* y, int accumulate, void* ws, cudaStream_t st,
                                 int passes, int act_bf16) {
  const int64_t n_loc = plan.expert_end - plan.expert_begin;
  int* work = static_cast<int*>(ws);
  if (cudaMemsetAsync(work, 0, 64 * sizeof(int), st) != cudaSuccess) {
    set_error("expert_fwd: memset failed");
    return OMNIMOE_ERR_CUDA;
  }
  const int32_t* m_loc = plan.expert_offsets + n_loc;
  const int d = (int)dm.d;
  omnimoe_status s = OMNIMOE_OK;
  if (!(passes & 1)) {
  } else if (resolve_group_size(dm) == 1 && d % 512 == 0 && d <= 2048) {
    // 32-byte loads, 80 registers (3 CTAs per SM), two x rows in flight: C3a pass Z 2.26 -> 2.17 ms
    // against 16-byte loads (<4,3,2> 2.17, <4,4,2> 2.21, <4,2,3> 2.29; profiles/r2/slices128/)
    auto go = [&](auto kern) {
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
      kern<<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(
          d, static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(W), plan.expert_offsets,
          plan.active, plan.n_active, plan.sorted_token, plan.sorted_gate, plan.sorted_task, plan.task_pair, dm.act,
          work);
    };
    switch (d / 512) {
      case 1: go(expert_zdot256_kernel<1, 3, 2>); break;
      case 2: go(expert_zdot256_kernel<2, 3, 2>); break;
      case 3: go(expert_zdot256_kernel<3, 3, 2>); break;
      default: go(expert_zdot256_kernel<4, 3, 2>); break;
    }
    OMNI_CHECK_LAUNCH("expert_zdot256_kernel");
  } else if (resolve_group_size(dm) == 1) {  // expert-major plan: w_e in registers, x from L2
    switch ((d + 255) / 256) {
      case 1: s = launch_zdot<1>(d, x, W, plan, dm.act, work, st); break;
      case 2: s = launch_zdot<2>(d, x, W, plan, dm.act, work, st); break;
      case 3: s = launch_zdot<3>(d, x, W, plan, dm.act, work, st); break;
      case 4: s = launch_zdot<4>(d, x, W, plan, dm.act, work, st); break;
      case 5: s = launch_zdot<5>(d, x, W, plan, dm.act, work, st); break;
      case 6: s = launch_zdot<6>(d, x, W, plan, dm.act, work, st); break;
      case 7: s = launch_zdot<7>(d, x, W, plan, dm.act, work, st); break;
      default: s = launch_zdot<8>(d, x, W, plan, dm.act, work, st); break;
    }
  } else switch ((d + 255) / 256) {
    case 1: s = launch_dot<1>(d, x, W, plan, m_loc, dm.act, work, st); break;
    case 2: s = launch_dot<2>(d, x, W, plan, m_loc, dm.act, work, st); break;
    case 3: s = launch_dot<3>(d, x, W, plan, m_loc, dm.act, work, st); break;
    case 4: s = launch_dot<4>(d, x, W, plan, m_loc, dm.act, work, st); break;
    case 5: s = launch_dot<5>(d, x, W, plan, m_loc, dm.act, work, st); break;
    case 6: s = launch_dot<6>(d, x, W, plan, m_loc, dm.act, work, st); break;
    case 7: s = launch_dot<7>(d, x, W, plan, m_loc, dm.act, work, st); break;
    default: s = launch_dot<8>(d, x, W, plan, m_loc, dm.act, work, st); break;
  }
  OMNI_TRY(s);
  if (!(passes & 2)) return OMNIMOE_OK;
  // 3 CTAs per SM; rounds of 8 tasks per window: 5 for the FHFMA (bf16 a) variant (C3a layer
  // 7.32 -> 7.18 ms, C5 42.0 -> 41.4 vs 4 rounds; profiles/r2/vconfig/), 4 for the FFMA2
  // variant (C3a pass V: <3,4> 2.82 ms, <4,4> 2.92, <3,6> 2.96, <2,8> 3.12; profiles/r2/slices128/)
  auto vkern = act_bf16 ? expert_vslice_kernel<3, 5, true> : expert_vslice_kernel<3, 4, false>;
#ifdef OMNIMOE_MEASURE
  switch (tuning().v_config) {  // (CTAs per SM, rounds of 8 tasks per window) sweep
    case 1: vkern = act_bf16 ? expert_vslice_kernel<4, 4, true> : expert_vslice_kernel<4, 4, false>; break;
    case 2: vkern = act_bf16 ? expert_vslice_kernel<3, 6, true> : expert_vslice_kernel<3, 6, false>; break;
    case 3: vkern = act_bf16 ? expert_vslice_kernel<2, 8, true> : expert_vslice_kernel<2, 8, false>; break;
    case 4: vkern = act_bf16 ? expert_vslice_kernel<4, 3, true> : expert_vslice_kernel<4, 3, false>; break;
    case 5: vkern = act_bf16 ? expert_vslice_kernel<3, 4, true> : expert_vslice_kernel<3, 5, false>; break;
    case 6: vkern = act_bf16 ? expert_vslice_kernel<4, 5, true> : expert_vslice_kernel<4, 5, false>; break;
    default: break;
  }
#endif
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, vkern, 256, 0);
  const int64_t n_tok = plan.n_tokens > 0 ? plan.n_tokens : L;
  const int nb = (int)resolve_v_bands(dm, n_loc, std::max<int64_t>(n_tok, 1));
  // one launch per expert band: its slices of V stay L2-resident while all tokens
  // use them; band b > 0 adds to the slices band b - 1 wrote (stream order: the
  // summation order is fixed, the result bitwise deterministic)
  // few tasks per token: 8 tokens per warp (lane groups), else one token per warp
  const bool grouped = dm.n_heads * dm.top_k <= tuning().v_group_max_tasks;
  int gper_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gper_sm, expert_vslice_group_kernel, 256, 0);
  for (int b = 0; b < nb; ++b) {
    if (grouped) {
      expert_vslice_group_kernel<<<num_sms() * std::max(gper_sm, 1), 256, 0, st>>>(
          d, L, n_loc, plan.token_offsets, nb + 1, b, n_tok, plan.task_pair, static_cast<const __nv_bfloat16*>(Vs),
          y, b > 0 ? 1 : accumulate, work + 1 + b);
      OMNI_CHECK_LAUNCH("expert_vslice_group_kernel");
    } else {
      vkern<<<num_sms() * per_sm, 256, 0, st>>>(
          d, L, n_loc, plan.token_offsets, nb + 1, b, n_tok, plan.task_pair, static_cast<const __nv_bfloat16*>(Vs),
          y, b > 0 ? 1 : accumulate, work + 1 + b);
      OMNI_CHECK_LAUNCH("expert_vslice_kernel");
    }
  }
  return OMNIMOE_OK;
}

omnimoe_status pack_v(int64_t n, int d, const void* V, void* Vs, cudaStream_t st) {
  if (n == 0) return OMNIMOE_OK;
  pack_v_kernel<<<num_sms() * 8, 256, 0, st>>>(static_cast<const uint4*>(V), static_cast<uint4*>(Vs), n, d);
  OMNI_CHECK_LAUNCH("pack_v_kernel");
  return OMNIMOE_OK;
}

// ---------------------------------------------------------------------------
// N2, d % 512 == 0: the routed-branch backward as row-gather passes, each holding at most
// one weight row per warp in registers (the fused two-warps-per-expert kernel above waits
// on a named barrier per task and runs at ~4 TB/s of L2 traffic):
//   1. z_p = x_l . w_e and q_p = dy_l . v_e for every plan position p (expert-major, the
//      pass-Z kernel shape: warp per active expert, weight row in registers, two gathered
//      rows in flight);
//   2. per p: s = sigma(z), dgate[t] = s q, dz = g q sigma'(z) (also into task_pair for the
//      dx pass), the coefficients dz and g s of the weight gradients;
//   3. dW_e = sum_p dz_p x_l and dV_e = sum_p g_p s_p dy_l: one warp per (active expert,
//      512-column part), fp32 accumulators in registers, the expert's rows gathered in plan
//      order (fixed summation order, no atomics);
//   4. dx (the SLICED pass V over the sliced W with a = dz), as before.
template <int NV8>
__global__ void __launch_bounds__(256, 3)
    expert_rowdot_kernel(int d, const __nv_bfloat16* __restrict__ rows, const __nv_bfloat16* __restrict__ Wt,
                         const int32_t* __restrict__ offsets, const int32_t* __restrict__ active,
                         const int32_t* __restrict__ n_active, const int32_t* __restrict__ stok,
                         float* __restrict__ out, int* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  const int na = *n_active;
  const uint64_t pol = policy_evict_first(), rpol = policy_evict_normal();
  int tau = 0;
  if (lane == 0) tau = atomicAdd(work, 1);
  tau = __shfl_sync(0xffffffffu, tau, 0);
  while (tau < na) {
    const int e = active[tau];
    const int beg = offsets[e], end = offsets[e + 1];
    U8 wv[NV8];
#pragma unroll
    for (int j = 0; j < NV8; ++j) wv[j] = ld256_hint(Wt + (size_t)e * d + (j * 32 + lane) * 16, pol);
    int nxt = 0;
    if (lane == 0) nxt = atomicAdd(work, 1);
    for (int p0 = beg; p0 < end; p0 += 32) {
      const int pl = p0 + lane;
      const int l_l = pl < end ? stok[pl] : 0;
      const int cnt = min(32, end - p0);
      float mine = 0.f;
      for (int t = 0; t < cnt; t += 2) {
        U8 xr[2][NV8];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int lt = __shfl_sync(0xffffffffu, l_l, min(t + u, cnt - 1));
#pragma unroll
          for (int j = 0; j < NV8; ++j) xr[u][j] = ld256_hint(rows + (size_t)lt * d + (j * 32 + lane) * 16, rpol);
        }
        float z[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          z[u] = 0.f;
#pragma unroll
          for (int j = 0; j < NV8; ++j) {
            float q = 0.f, q2 = 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              q = dot2_bf16(q, wv[j].w[i], xr[u][j].w[i]);
              q2 = dot2_bf16(q2, wv[j].w[4 + i], xr[u][j].w[4 + i]);
            }
            z[u] += q + q2;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < 2; ++u) z[u] += __shfl_xor_sync(0xffffffffu, z[u], o);
        if (lane == t) mine = z[0];
        if (lane == t + 1) mine = z[1];
      }
      if (lane < cnt) out[pl] = mine;
    }
    tau = __shfl_sync(0xffffffffu, nxt, 0);
  }
}

__global__ void bwd_scalars_kernel(const int32_t* __restrict__ m_loc_p, const float* __restrict__ zb,
                                   const float* __restrict__ qb, const float* __restrict__ sgate,
                                   const int32_t* __restrict__ stask, float* __restrict__ dgate,
                                   int32_t* __restrict__ task_pair, float* __restrict__ cw, float* __restrict__ cv,
                                   int act) {
  const int64_t m = *m_loc_p;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    const float z = zb[p], q = qb[p], g = sgate[p];
    const float lg = 1.0f / (1.0f + __expf(-z));
    const float sz = act == OMNIMOE_IDENTITY ? z : z * lg;
    const float sp = act == OMNIMOE_IDENTITY ? 1.0f : lg * (1.0f + z * (1.0f - lg));
    const float dz = g * q * sp;
    const int t = stask[p];
    dgate[t] = sz * q;
    task_pair[2 * (size_t)t + 1] = __float_as_int(dz);
    cw[p] = dz;
    cv[p] = g * sz;
  }
}

// out[tau][part] = sum over the expert's plan positions p of coef[p] * rows[tok[p]][part]:
// one warp per (active expert, part of PW x 512 columns), T rows in flight.  Items hold
// ~eta tasks, so the next item is claimed and its expert / segment looked up while the
// current item's rows are in flight (the item-to-item dependency chain is the cost).
template <int T, int PW, int MINB>
__global__ void __launch_bounds__(256, MINB)
    expert_accum_kernel(int d, const __nv_bfloat16* __restrict__ rows, const float* __restrict__ coef,
                        const int32_t* __restrict__ offsets, const int32_t* __restrict__ active,
                        const int32_t* __restrict__ n_active, const int32_t* __restrict__ stok,
                        float* __restrict__ out, int* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  const int parts = d / (512 * PW);  // 16 PW columns per lane and part
  const int64_t n_items = (int64_t)(*n_active) * parts;
  auto claim = [&]() {
    int v = 0;
    if (lane == 0) v = atomicAdd(work, 1);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  auto meta = [&](int64_t item, int& beg, int& end) {
    beg = end = 0;
    if (item < n_items) {
      const int e = active[item / parts];
      beg = offsets[e];
      end = offsets[e + 1];
    }
  };
  int64_t it = claim();
  int beg, end;
  meta(it, beg, end);
  while (it < n_items) {
    const int tau = (int)(it / parts), part = (int)(it - (int64_t)tau * parts);
    const int col = part * 512 * PW + lane * 16;
    const int64_t nxt = claim();  // in flight while this item's rows are
    unsigned long long acc[PW][8];
#pragma unroll
    for (int j = 0; j < PW; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[j][i] = 0ull;
    int nbeg = 0, nend = 0;
    bool fetched = false;
    for (int p0 = beg; p0 < end; p0 += 32) {
      const int pl = p0 + lane;
      const int l_l = pl < end ? stok[pl] : 0;
      const float c_l = pl < end ? coef[pl] : 0.f;
      const int cnt = min(32, end - p0);
      for (int t = 0; t < cnt; t += T) {
        U8 r[T][PW];
        float c[T];
#pragma unroll
        for (int u = 0; u < T; ++u) {
          const int src = min(t + u, cnt - 1);
          const int l = __shfl_sync(0xffffffffu, l_l, src);
          c[u] = t + u < cnt ? __shfl_sync(0xffffffffu, c_l, src) : 0.f;
#pragma unroll
          for (int j = 0; j < PW; ++j) r[u][j] = ld256(rows + (size_t)l * d + col + j * 512);
        }
        if (!fetched) {  // the next item's segment, behind this item's first row loads
          meta(nxt, nbeg, nend);
          fetched = true;
        }
#pragma unroll
        for (int u = 0; u < T; ++u) {
          const unsigned long long c2 = ((unsigned long long)__float_as_uint(c[u]) << 32) | __float_as_uint(c[u]);
#pragma unroll
          for (int j = 0; j < PW; ++j)
#pragma unroll
            for (int i = 0; i < 8; ++i) axpy2_bf16(acc[j][i], c2, r[u][j].w[i]);
        }
      }
    }
    if (!fetched) meta(nxt, nbeg, nend);
#pragma unroll
    for (int j = 0; j < PW; ++j) {
      float4* dst = reinterpret_cast<float4*>(out + (size_t)tau * d + col + j * 512);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        dst[q] = make_float4(lo_f(acc[j][2 * q]), hi_f(acc[j][2 * q]), lo_f(acc[j][2 * q + 1]),
                             hi_f(acc[j][2 * q + 1]));
    }
    it = nxt;
    beg = nbeg;
    end = nend;
  }
}

omnimoe_status expert_bwd_run(const omnimoe_dims& dm, int64_t L, const void* x, const void* W, const void* V,
                              const void* Ws, const omnimoe_plan& plan, const void* dy, float* dx, float* dW_act,
                              float* dV_act, float* dgate, int accumulate_dx, void* ws, cudaStream_t st) {
  const int d = (int)dm.d;
  // row-gather passes (above) when experts are shared (eta >= 2; C3a 19.2 -> 16.3 ms); at
  // eta ~ 1 every expert has ~one task and the fused kernel's single gather of x and dy per
  // task wins (C3b 1.6 vs 2.6 ms)
  if (d % 512 == 0 && d <= 2048 && expected_eta(dm, L) >= 2.0) {
    const int64_t n_loc = plan.expert_end - plan.expert_begin;
    const int64_t M = bwd_ws_tasks(dm, L);
    int* work = static_cast<int*>(ws);
    float* zb = reinterpret_cast<float*>(static_cast<char*>(ws) + 256);
    float* qb = zb + M;
    float* cw = qb + M;
    float* cv = cw + M;
    if (cudaMemsetAsync(work, 0, 64 * sizeof(int), st) != cudaSuccess) {
      set_error("expert_bwd: memset failed");
      return OMNIMOE_ERR_CUDA;
    }
    auto X = static_cast<const __nv_bfloat16*>(x);
    auto D = static_cast<const __nv_bfloat16*>(dy);
    auto Wp = static_cast<const __nv_bfloat16*>(W);
    auto Vp = static_cast<const __nv_bfloat16*>(V);
    auto rowdot = [&](const __nv_bfloat16* rows, const __nv_bfloat16* Wt, float* out, int* w) {
      auto go = [&](auto kern) {
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        kern<<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(d, rows, Wt, plan.expert_offsets, plan.active,
                                                               plan.n_active, plan.sorted_token, out, w);
      };
      switch (d / 512) {
        case 1: go(expert_rowdot_kernel<1>); break;
        case 2: go(expert_rowdot_kernel<2>); break;
        case 3: go(expert_rowdot_kernel<3>); break;
        default: go(expert_rowdot_kernel<4>); break;
      }
    };
    rowdot(X, Wp, zb, work);
    OMNI_CHECK_LAUNCH("expert_rowdot_kernel(z)");
    rowdot(D, Vp, qb, work + 1);
    OMNI_CHECK_LAUNCH("expert_rowdot_kernel(q)");
    const int32_t* m_loc = plan.expert_offsets + n_loc;
    bwd_scalars_kernel<<<num_sms() * 8, 256, 0, st>>>(m_loc, zb, qb, plan.sorted_gate, plan.sorted_task, dgate,
                                                     plan.task_pair, cw, cv, dm.act);
    OMNI_CHECK_LAUNCH("bwd_scalars_kernel");
    auto accum = [&](const __nv_bfloat16* rows, const float* coef, float* out, int* w) {
      auto go = [&](auto kern) {
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        kern<<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(d, rows, coef, plan.expert_offsets, plan.active,
                                                               plan.n_active, plan.sorted_token, out, w);
      };
      // C3a, both weight gradients: <4 rows, 1024 columns, 2 CTAs> 8.1 ms, <4, 512, 3> 8.8,
      // <8, 512, 2> 10.6, <8, 512, 3> 12.1 (the fp32 dW / dV rows are 17 GB of writes)
      if (d % 1024 == 0) go(expert_accum_kernel<4, 2, 2>);
      else go(expert_accum_kernel<4, 1, 3>);
    };
    accum(X, cw, dW_act, work + 2);
    OMNI_CHECK_LAUNCH("expert_accum_kernel(dW)");
    accum(D, cv, dV_act, work + 3);
    OMNI_CHECK_LAUNCH("expert_accum_kernel(dV)");
    omnimoe_dims dv = dm;
    dv.v_layout = OMNIMOE_V_SLICED;
    return expert_sliced_run(dv, L, x, W, Ws, plan, dx, accumulate_dx, static_cast<char*>(ws) + 256 + 16 * M, st,
                             2, /*act_bf16=*/0);
  }
  // d >= 1024: four warps per expert (a quarter of the columns each: more warps resident),
  // else a pair
  const bool quad = d >= 1024;
  const int nvh = (d / (quad ? 4 : 2) + 255) / 256;
  int per_sm = 1;
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto Wp = static_cast<const __nv_bfloat16*>(W);
  auto Vp = static_cast<const __nv_bfloat16*>(V);
  auto D = static_cast<const __nv_bfloat16*>(dy);
#define OMNI_BWD_CASE(N, G)                                                                                     \
  {                                                                                                            \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expert_bwd_kernel<N, G>, 256, 0);                   \
    expert_bwd_kernel<N, G><<<num_sms() * std::max(per_sm, 1), 256, 0, st>>>(                                       \
        d, X, Wp, Vp, D, plan.expert_offsets, plan.active, plan.n_active, plan.sorted_token, plan.sorted_gate, \
        plan.sorted_task, plan.task_pair, dgate, dW_act, dV_act, dm.act);                                      \
  }
  if (quad) {
    if (nvh <= 1) OMNI_BWD_CASE(1, 4) else OMNI_BWD_CASE(2, 4)
  } else {
    if (nvh <= 1) OMNI_BWD_CASE(1, 2) else OMNI_BWD_CASE(2, 2)
  }
#undef OMNI_BWD_CASE
  OMNI_CHECK_LAUNCH("expert_bwd_kernel");
  // dx_l = sum_t dz_t w_e: the token-stationary slice pass over the sliced W
  omnimoe_dims dv = dm;
  dv.v_layout = OMNIMOE_V_SLICED;
  return expert_sliced_run(dv, L, x, W, Ws, plan, dx, accumulate_dx, ws, st, 2, /*act_bf16=*/0);
}

omnimoe_status expert_run(const omnimoe_dims& dm, int64_t L, const void* x, const void* W,
                          const void* V, const omnimoe_plan& plan, float* y, int accumulate,
                          void* ws, cudaStream_t st, int act_bf16) {
  if (dm.v_layout == OMNIMOE_V_SLICED)
    return expert_sliced_run(dm, L, x, W, V, plan, y, accumulate, ws, st, 3, act_bf16);
  if (!accumulate) {
    if (cudaMemsetAsync(y, 0, (size_t)L * dm.d * sizeof(float), st) != cudaSuccess) {
      set_error("expert_fwd: memset failed");
      return OMNIMOE_ERR_CUDA;
    }
  }
  const int64_t B = resolve_group_size(dm);
  const int64_t n_loc = plan.expert_end - plan.expert_begin;
  if (B > 1) {
    int* work = static_cast<int*>(ws);
    if (cudaMemsetAsync(work, 0, sizeof(int), st) != cudaSuccess) {
      set_error("expert_fwd: memset failed");
      return OMNIMOE_ERR_CUDA;
    }
    if (dm.dtype == OMNIMOE_BF16)
      return launch_group<__nv_bfloat16>((int)dm.d, x, W, V, plan, n_loc, y, dm.act, work, st);
    return launch_group<float>((int)dm.d, x, W, V, plan, n_loc, y, dm.act, work, st);
  }
  if (dm.dtype == OMNIMOE_BF16) return launch_warp<__nv_bfloat16>((int)dm.d, x, W, V, plan, y, dm.act, st);
  return launch_warp<float>((int)dm.d, x, W, V, plan, y, dm.act, st);
}

}  // namespace omni
