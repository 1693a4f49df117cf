// ============================================================================
// OmniMoE layer-forward ORACLE -- test infrastructure, NOT the product.
//
// Plain, slow, obviously-correct CPU implementation (C++17, fp64) of what the
// OmniMoE atomic-expert layer forward computes (arXiv 2602.05711, PAPER.md).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this library.  It shares no code, header or
// constant with the CUDA path (paper_2602_05711_b200/csrc) and includes no
// CUDA header.
//
// Citations: "PAPER:n" = /root/reference/PAPER.md line n (section / equation
// named alongside); "Q#" = a reading listed in DESIGN.md "Readings".
//
// Pins: every function below is pinned by tests/test_oracle.py (-m "not gpu")
// against closed forms, brute force, invariants and SPEC worked examples.
// Absolute layer outputs at paper scale (the paper prints none, P12)
// are pinned by closed forms at d = 2048, K = 512 (constant expert rows:
// y = h silu(x.w) u for any routing; one-hot expert rows: the gate-weighted
// scatter of the selected ids) -- test_layer_closed_forms_paper_width.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

namespace {

// --------------------------------------------------------------------------
// Exact key of a grid cell: the exact real s_r[i] + s_c[j] (Eq.S, PAPER:220-224,
// ranked on raw logits per reading Q8), represented as the TwoSum pair
// (hi, lo): hi = RN64(s_r + s_c), lo = exact residual.  Lexicographic order on
// (hi, lo) is the order of the exact reals.  Ties between EXACTLY equal keys
// go to the smaller flat id n = i*N_c + j (reading Q7).
// --------------------------------------------------------------------------
struct Key {
  double hi, lo;
  int64_t n;  // flat expert id
};

inline Key make_key(float sr, float sc, int64_t n) {
  double a = (double)sr, b = (double)sc;
  double hi = a + b;
  double bb = hi - a;
  double lo = (a - (hi - bb)) + (b - bb);  // Knuth TwoSum: exact residual
  return Key{hi, lo, n};
}

// true iff p precedes q in the total order (larger exact key first, then
// smaller flat id).
inline bool precedes(const Key& p, const Key& q) {
  if (p.hi != q.hi) return p.hi > q.hi;
  if (p.lo != q.lo) return p.lo > q.lo;
  return p.n < q.n;
}

// --------------------------------------------------------------------------
// Exact dot product of fp32-representable values, rounded ONCE to fp32 with
// round-to-nearest-even (reading Q9: "scores computed in fp32 from
// bf16-rounded inputs" = RN32 of the real dot product).  Every input is an
// integer mantissa m (|m| < 2^24) times 2^e, so every product is an integer
// (< 2^48) times 2^(e1+e2); the products are summed exactly in a 128-bit
// integer at the smallest product exponent, then rounded to 24 significant
// bits.  Inputs that are not fp32 values, or whose product exponents spread
// beyond the 128-bit accumulator, give NaN (never the case for bf16/fp32
// tensors of the synthetic generator; tests/test_oracle.py checks the NaN).
// --------------------------------------------------------------------------
struct Dyadic {
  int64_t m;  // odd or zero
  int e;
  bool ok;    // false: not an fp32-representable value
};

inline Dyadic to_dyadic(double v) {
  if (v == 0.0) return Dyadic{0, 0, true};
  if (!std::isfinite(v)) return Dyadic{0, 0, false};
  int ex;
  double f = std::frexp(v, &ex);                 // v = f * 2^ex, 0.5 <= |f| < 1
  int64_t m = (int64_t)std::ldexp(f, 53);        // exact: v has <= 53 significant bits
  int e = ex - 53;
  while ((m & 1) == 0) { m /= 2; ++e; }
  return Dyadic{m, e, m < (int64_t(1) << 24) && m > -(int64_t(1) << 24)};
}

inline float round_int128_to_f32(__int128 S, int e) {  // RN32(S * 2^e)
  if (S == 0) return 0.0f;
  const bool neg = S < 0;
  unsigned __int128 a = neg ? (unsigned __int128)(-S) : (unsigned __int128)S;
  int msb = 127;
  while (!((a >> msb) & 1)) --msb;
  if (msb > 23) {  // keep 24 significant bits, round half to even
    const int sh = msb - 23;
    unsigned __int128 q = a >> sh;
    unsigned __int128 rem = a - (q << sh);
    unsigned __int128 half = (unsigned __int128)1 << (sh - 1);
    if (rem > half || (rem == half && (q & 1))) q += 1;
    a = q;
    e += sh;
  }
  // a < 2^25 now: exact in double; scaling by 2^e is exact for normal fp32 results
  const double r = std::ldexp((double)(uint64_t)a, e);
  return (float)(neg ? -r : r);
}

inline float exact_dot_rn32(const double* x, const double* w, int64_t d) {
  std::vector<Dyadic> p;
  p.reserve(d);
  int emin = 1 << 30;
  for (int64_t k = 0; k < d; ++k) {
    Dyadic a = to_dyadic(x[k]), b = to_dyadic(w[k]);
    if (!a.ok || !b.ok) return NAN;
    if (a.m == 0 || b.m == 0) continue;
    Dyadic q{a.m * b.m, a.e + b.e, true};
    emin = std::min(emin, q.e);
    p.push_back(q);
  }
  __int128 S = 0;
  for (const Dyadic& q : p) {
    const int sh = q.e - emin;
    int bits = 0;
    for (uint64_t a = (uint64_t)(q.m < 0 ? -q.m : q.m); a; a >>= 1) ++bits;
    if (bits + sh > 126 - 20) return NAN;  // beyond the 128-bit accumulator (d <= 2^20)
    S += (__int128)q.m << sh;
  }
  return round_int128_to_f32(S, emin);
}

inline double silu(double z) { return z / (1.0 + std::exp(-z)); }  // reading Q1

inline double act_fn(double z, int act) { return act == 1 ? z : silu(z); }

template <class F>
void parallel_for(int64_t n, int nthreads, F f) {
  if (nthreads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t b = t * chunk, e = std::min<int64_t>(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([=]() { for (int64_t i = b; i < e; ++i) f(i); });
  }
  for (auto& t : th) t.join();
}

// Per-token-head routing result in the order of the total order above.
struct RouteOut {
  std::vector<Key> top;  // first min(K+1, N) keys
};

// O3 brute force (Eq.TopK): score every one of the N grid
// cells, order all of them, keep the first K+1 (the extra one gives the gap).
void select_bruteforce(const float* sr, int64_t Nr, const float* sc, int64_t Nc, int64_t K,
                       std::vector<Key>& out) {
  std::vector<Key> all;
  all.reserve(Nr * Nc);
  for (int64_t i = 0; i < Nr; ++i)
    for (int64_t j = 0; j < Nc; ++j) all.push_back(make_key(sr[i], sc[j], i * Nc + j));
  int64_t keep = std::min<int64_t>(K + 1, Nr * Nc);
  std::partial_sort(all.begin(), all.begin() + keep, all.end(), precedes);
  out.assign(all.begin(), all.begin() + keep);
}

// O4 product selection: order rows by (s_r desc, i asc) and columns by
// (s_c desc, j asc); a cell with 1-based ranks (a, b) has at least a*b - 1
// predecessors, so only cells with a*b <= K+1 can be among the first K+1
// (the north star's k x k candidate grid is a
// superset).  Candidates are ordered exactly like brute force.
void select_product(const float* sr, int64_t Nr, const float* sc, int64_t Nc, int64_t K,
                    std::vector<Key>& out) {
  std::vector<int64_t> ri(Nr), ci(Nc);
  std::iota(ri.begin(), ri.end(), 0);
  std::iota(ci.begin(), ci.end(), 0);
  std::sort(ri.begin(), ri.end(), [&](int64_t p, int64_t q) {
    return sr[p] != sr[q] ? sr[p] > sr[q] : p < q;
  });
  std::sort(ci.begin(), ci.end(), [&](int64_t p, int64_t q) {
    return sc[p] != sc[q] ? sc[p] > sc[q] : p < q;
  });
  int64_t K1 = K + 1;
  std::vector<Key> cand;
  for (int64_t a = 1; a <= std::min(K1, Nr); ++a)
    for (int64_t b = 1; b <= std::min(K1, Nc) && a * b <= K1; ++b) {
      int64_t i = ri[a - 1], j = ci[b - 1];
      cand.push_back(make_key(sr[i], sc[j], i * Nc + j));
    }
  int64_t keep = std::min<int64_t>(K1, Nr * Nc);
  std::partial_sort(cand.begin(), cand.begin() + keep, cand.end(), precedes);
  out.assign(cand.begin(), cand.begin() + keep);
}

// Paper App. A "Block-wise Merge Selection": partition the N
// flat ids into blocks of B_sel, score each block on the fly, take its local
// top by iterative max-reduction, merge into a running global top buffer by
// insertion.  Kept only as a cross-check of the two selectors above.
void select_blockmerge(const float* sr, int64_t Nr, const float* sc, int64_t Nc, int64_t K,
                       int64_t B_sel, std::vector<Key>& out) {
  int64_t N = Nr * Nc, K1 = std::min<int64_t>(K + 1, N);
  std::vector<Key> global;  // sorted by precedes, size <= K1
  for (int64_t b0 = 0; b0 < N; b0 += B_sel) {
    int64_t b1 = std::min(N, b0 + B_sel);
    std::vector<Key> blk;
    for (int64_t n = b0; n < b1; ++n) blk.push_back(make_key(sr[n / Nc], sc[n % Nc], n));
    std::vector<char> taken(blk.size(), 0);
    for (int64_t r = 0; r < std::min<int64_t>(K1, (int64_t)blk.size()); ++r) {  // iterative max
      int64_t best = -1;
      for (int64_t t = 0; t < (int64_t)blk.size(); ++t)
        if (!taken[t] && (best < 0 || precedes(blk[t], blk[best]))) best = t;
      taken[best] = 1;
      // insertion into the global buffer
      Key k = blk[best];
      auto pos = std::upper_bound(global.begin(), global.end(), k, precedes);
      global.insert(pos, k);
      if ((int64_t)global.size() > K1) global.pop_back();
    }
  }
  out = global;
}

}  // namespace

extern "C" {

// Load metrics of a routing decision (following PKM/PEER): with
// z_i = c_i / M the normalised retrieval frequency of expert i (c_i tasks, M
// tasks in total, N experts),
//   Expert Usage = |{i : z_i > 0}| / N
//   Unevenness   = D_KL(z || U) = sum_{i: z_i > 0} z_i log(N z_i).
// out[0] = usage, out[1] = unevenness (0, 0 when M = 0).
void oracle_load_stats(int64_t N, const int64_t* counts, double* out) {
  int64_t M = 0, used = 0;
  for (int64_t i = 0; i < N; ++i) {
    M += counts[i];
    used += counts[i] > 0;
  }
  double kl = 0.0;
  for (int64_t i = 0; i < N; ++i)
    if (counts[i] > 0) {
      const double z = (double)counts[i] / (double)M;
      kl += z * std::log((double)N * z);
    }
  out[0] = M > 0 ? (double)used / (double)N : 0.0;
  out[1] = M > 0 ? kl : 0.0;
}

// The ablation "w/o Cartesian Product Router": a dense routing
// projection scores every expert, s = x W_g (logits [T][N] fp32), and the
// router takes the exact top-K of the N scores by (value desc, id asc) (the
// tie rule of Q7), gates = softmax over the selected (Eq.Gate).
// Brute force: sort all N.  gap[t] = s_K - s_{K+1} (+inf when K == N).
void oracle_dense_route(int64_t T, int64_t N, int64_t K, const float* logits, int nthreads, int32_t* idx,
                        double* gate, double* key, double* gap) {
  parallel_for(T, nthreads, [&](int64_t t) {
    const float* s = logits + t * N;
    std::vector<int64_t> ord(N);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return s[a] > s[b]; });
    const double k1 = s[ord[0]];
    double den = 0.0;
    for (int64_t k = 0; k < K; ++k) den += std::exp((double)s[ord[k]] - k1);
    for (int64_t k = 0; k < K; ++k) {
      idx[t * K + k] = (int32_t)ord[k];
      key[t * K + k] = s[ord[k]];
      gate[t * K + k] = std::exp((double)s[ord[k]] - k1) / den;
    }
    gap[t] = K < N ? (double)s[ord[K - 1]] - (double)s[ord[K]] : INFINITY;
  });
}

// N2 (backward of the routed branch) for a fixed routing decision:
// y_l = sum_k g_lk sigma(z_lk) v_n,  z_lk = x_l . w_n,  n = ids[l][k]  (Eq.Assemble).
// Given dy = dLoss/dy (all fp64), the gradients follow the chain rule term by term:
//   q = dy_l . v_n,  dgate_lk = sigma(z) q,  dz = g q sigma'(z),
//   dV_n += g sigma(z) dy_l,  dW_n += dz x_l,  dx_l += dz w_n.
// sigma = SiLU (reading Q1): sigma'(z) = s(z) (1 + z (1 - s(z))), s = logistic; IDENTITY: 1.
// dW, dV: [rows][d] indexed like W, V (ids index their rows).
void oracle_routed_bwd(int64_t L, int64_t d, int64_t HK, const double* x, const double* W, const double* V,
                       const int32_t* ids, const double* gates, const double* dy, int act, int64_t rows,
                       double* dx, double* dW, double* dV, double* dgate) {
  std::fill(dx, dx + L * d, 0.0);
  std::fill(dW, dW + rows * d, 0.0);
  std::fill(dV, dV + rows * d, 0.0);
  for (int64_t l = 0; l < L; ++l)
    for (int64_t k = 0; k < HK; ++k) {
      const int64_t n = ids[l * HK + k];
      const double g = gates[l * HK + k];
      double z = 0.0, q = 0.0;
      for (int64_t c = 0; c < d; ++c) {
        z += x[l * d + c] * W[n * d + c];
        q += dy[l * d + c] * V[n * d + c];
      }
      const double lg = 1.0 / (1.0 + std::exp(-z));
      const double s = act ? z : z * lg;
      const double sp = act ? 1.0 : lg * (1.0 + z * (1.0 - lg));
      const double dz = g * q * sp;
      dgate[l * HK + k] = s * q;
      for (int64_t c = 0; c < d; ++c) {
        dV[n * d + c] += g * s * dy[l * d + c];
        dW[n * d + c] += dz * x[l * d + c];
        dx[l * d + c] += dz * W[n * d + c];
      }
    }
}

// N2, router part: gradients through Eq.Gate (softmax over the K selected keys,
// PAPER:136-139) and Eq.S / Eq.Logits (key = s_r[i] + s_c[j], s = x . sub, PAPER:
// 211-224) with the selection held fixed (top-K is piecewise constant).  Per token-
// head: dkappa_k = g_k (dgate_k - sum_j g_j dgate_j); ds_r[i] += dkappa, ds_c[j] +=
// dkappa; dsub[h][r] += ds[l][h][r] x_l; dx_l += sum_r ds[l][h][r] sub[h][r].
// gate: the forward gates; dx accumulates; dsub [h][Nr+Nc][d] is overwritten.
void oracle_router_bwd(int64_t L, int64_t d, int64_t h, int64_t Nr, int64_t Nc, int64_t K, const double* x,
                       const double* sub, const int32_t* idx, const double* gate, const double* dgate, double* dx,
                       double* dsub) {
  const int64_t R = Nr + Nc;
  std::fill(dsub, dsub + h * R * d, 0.0);
  std::vector<double> ds(R);
  for (int64_t l = 0; l < L; ++l)
    for (int64_t hh = 0; hh < h; ++hh) {
      const int64_t t = l * h + hh;
      double dot = 0.0;
      for (int64_t k = 0; k < K; ++k) dot += gate[t * K + k] * dgate[t * K + k];
      std::fill(ds.begin(), ds.end(), 0.0);
      for (int64_t k = 0; k < K; ++k) {
        const double dk = gate[t * K + k] * (dgate[t * K + k] - dot);
        const int64_t n = idx[t * K + k];
        ds[n / Nc] += dk;
        ds[Nr + n % Nc] += dk;
      }
      for (int64_t r = 0; r < R; ++r) {
        if (ds[r] == 0.0) continue;
        const double* sr = sub + (hh * R + r) * d;
        double* dr = dsub + (hh * R + r) * d;
        for (int64_t c = 0; c < d; ++c) {
          dr[c] += ds[r] * x[l * d + c];
          dx[l * d + c] += ds[r] * sr[c];
        }
      }
    }
}

// N2, shared MLP (reading Q2): G = x W_g^T, U = x W_u^T, H = SiLU(G) U, y = H W_down^T.
// dH = dy W_down; dU = dH SiLU(G); dG = dH U SiLU'(G); dW_down = dy^T H;
// dW_gu = [dG dU]^T x (gate rows then up rows); dx += dG W_g + dU W_u.
void oracle_mlp_bwd(int64_t L, int64_t d, int64_t dff, const double* x, const double* w_gu, const double* w_down,
                    const double* dy, double* dx, double* dw_gu, double* dw_down) {
  std::fill(dw_gu, dw_gu + 2 * dff * d, 0.0);
  std::fill(dw_down, dw_down + d * dff, 0.0);
  std::vector<double> G(dff), U(dff), H(dff), dH(dff);
  for (int64_t l = 0; l < L; ++l) {
    const double* xl = x + l * d;
    const double* gl = dy + l * d;
    for (int64_t f = 0; f < dff; ++f) {
      double g = 0.0, u = 0.0;
      for (int64_t c = 0; c < d; ++c) {
        g += xl[c] * w_gu[f * d + c];
        u += xl[c] * w_gu[(dff + f) * d + c];
      }
      G[f] = g;
      U[f] = u;
      H[f] = g / (1.0 + std::exp(-g)) * u;
      double s = 0.0;
      for (int64_t c = 0; c < d; ++c) s += gl[c] * w_down[c * dff + f];
      dH[f] = s;
    }
    for (int64_t c = 0; c < d; ++c)
      for (int64_t f = 0; f < dff; ++f) dw_down[c * dff + f] += gl[c] * H[f];
    for (int64_t f = 0; f < dff; ++f) {
      const double sg = 1.0 / (1.0 + std::exp(-G[f]));
      const double silu = G[f] * sg, dsilu = sg * (1.0 + G[f] * (1.0 - sg));
      const double dU = dH[f] * silu, dG = dH[f] * U[f] * dsilu;
      for (int64_t c = 0; c < d; ++c) {
        dw_gu[f * d + c] += dG * xl[c];
        dw_gu[(dff + f) * d + c] += dU * xl[c];
        dx[l * d + c] += dG * w_gu[f * d + c] + dU * w_gu[(dff + f) * d + c];
      }
    }
  }
}

// O1 logits (Eq.Logits; reading Q9): for each token l, head h
// and sub-key row r (rows [0,N_r) are W_r's columns, rows [N_r, N_r+N_c) are
// W_c's), s = RN32(sum_k x[l][k]*sub[h][r][k]) -- the fp32 round-to-nearest-
// even of the EXACT real dot product (exact_dot_rn32 above).
// The same function as exact_dot_rn32 per (token, head, row), organised for
// speed: every row is written ONCE as integers at the row's finest exponent,
// v_k = M_k * 2^E_row (exact; M_k = m_k * 2^(e_k - E_row)), so that a dot
// product is sum_k Mx_k * Mw_k (exact in a 128-bit integer) times
// 2^(E_x + E_w), rounded once (round_int128_to_f32).  A row whose integers do
// not fit 62 bits, or a pair whose products could exceed the accumulator, is
// left to exact_dot_rn32 (tests/test_oracle.py::test_logits_row_integer_path
// checks both routes against Python Fractions).
struct IntRow {
  std::vector<int64_t> M;
  int E = 0;
  int bits = 0;     // bits of max |M_k|
  bool ok = false;  // false: use exact_dot_rn32
};

inline IntRow int_row(const double* v, int64_t d) {
  IntRow r;
  std::vector<Dyadic> q(d);
  int emin = 1 << 30;
  for (int64_t k = 0; k < d; ++k) {
    q[k] = to_dyadic(v[k]);
    if (!q[k].ok) return r;
    if (q[k].m != 0) emin = std::min(emin, q[k].e);
  }
  r.M.assign(d, 0);
  r.E = emin == (1 << 30) ? 0 : emin;
  uint64_t amax = 0;
  for (int64_t k = 0; k < d; ++k) {
    if (q[k].m == 0) continue;
    const int sh = q[k].e - r.E;
    const uint64_t a = (uint64_t)(q[k].m < 0 ? -q[k].m : q[k].m);
    int b = 0;
    for (uint64_t t = a; t; t >>= 1) ++b;
    if (b + sh > 62) return r;  // r.ok stays false
    r.M[k] = q[k].m * ((int64_t)1 << sh);
    amax = std::max(amax, a << sh);
  }
  for (uint64_t t = amax; t; t >>= 1) ++r.bits;
  r.ok = true;
  return r;
}

void oracle_logits(int64_t L, int64_t d, int64_t h, int64_t R, const double* x, const double* sub,
                   float* out, int nthreads) {
  std::vector<IntRow> wrow(h * R);
  parallel_for(h * R, nthreads, [&](int64_t r) { wrow[r] = int_row(sub + r * d, d); });
  int lg = 0;
  while (((int64_t)1 << lg) < d) ++lg;
  const int64_t TB = 16;  // tokens per block: each sub-key row is read once per block
  parallel_for((L + TB - 1) / TB, nthreads, [&](int64_t blk) {
    const int64_t l0 = blk * TB, l1 = std::min(L, l0 + TB);
    std::vector<IntRow> xr(l1 - l0);
    for (int64_t l = l0; l < l1; ++l) xr[l - l0] = int_row(x + l * d, d);
    for (int64_t hh = 0; hh < h; ++hh)
      for (int64_t r = 0; r < R; ++r) {
        const IntRow& wr = wrow[hh * R + r];
        for (int64_t l = l0; l < l1; ++l) {
          const IntRow& xl = xr[l - l0];
          float& o = out[(l * h + hh) * R + r];
          if (!xl.ok || !wr.ok || xl.bits + wr.bits + lg > 125) {
            o = exact_dot_rn32(x + l * d, sub + (hh * R + r) * d, d);
            continue;
          }
          __int128 S = 0;
          if (xl.bits + wr.bits + lg <= 62) {  // every partial sum fits int64
            int64_t s64 = 0;
            for (int64_t k = 0; k < d; ++k) s64 += xl.M[k] * wr.M[k];
            S = s64;
          } else {
            for (int64_t k = 0; k < d; ++k) S += (__int128)xl.M[k] * wr.M[k];
          }
          o = round_int128_to_f32(S, xl.E + wr.E);
        }
      }
  });
}

// Exact dot product rounded once to fp32, exported for the pins.
float oracle_exact_dot(const double* x, const double* w, int64_t d) { return exact_dot_rn32(x, w, d); }

// O2-O5 routing for a batch of token-heads (Eq.TopK + Eq.Gate, PAPER:131-139;
// Eq.S).  logits: [T][N_r + N_c] fp32 (T = L*h token-heads).
// method: 0 brute force, 1 product, 2 block-merge (B_sel = bsel).
// Outputs per token-head t (K entries in the total order):
//   idx[t][k]    flat expert id
//   gate[t][k]   g_k = exp(kappa_k - kappa_1) / sum_k' exp(kappa_k' - kappa_1)
//                (softmax over the selected keys only; Q11)
//   score[t][k]  kappa_k - lse_r - lse_c = p_r[i] + p_c[j] (Eq.LSM + Eq.S; Q8)
//   key_hi/key_lo[t][k] exact key pair, gap[t] = kappa_K - kappa_{K+1}
//                (+inf when K == N)
void oracle_route(int64_t T, int64_t Nr, int64_t Nc, int64_t K, const float* logits, int method,
                  int64_t bsel, int nthreads, int32_t* idx, double* gate, double* score,
                  double* key_hi, double* key_lo, double* gap) {
  int64_t R = Nr + Nc;
  parallel_for(T, nthreads, [&](int64_t t) {
    const float* sr = logits + t * R;
    const float* sc = sr + Nr;
    std::vector<Key> top;
    if (method == 0) select_bruteforce(sr, Nr, sc, Nc, K, top);
    else if (method == 1) select_product(sr, Nr, sc, Nc, K, top);
    else select_blockmerge(sr, Nr, sc, Nc, K, bsel, top);
    // log-sum-exp per half (Eq.LSM)
    auto lse = [](const float* s, int64_t n) {
      double m = -INFINITY;
      for (int64_t i = 0; i < n; ++i) m = std::max(m, (double)s[i]);
      double acc = 0.0;
      for (int64_t i = 0; i < n; ++i) acc += std::exp((double)s[i] - m);
      return m + std::log(acc);
    };
    double lr = lse(sr, Nr), lc = lse(sc, Nc);
    double k1 = top[0].hi + top[0].lo;
    double den = 0.0;
    for (int64_t k = 0; k < K; ++k) den += std::exp((top[k].hi - k1) + top[k].lo);
    for (int64_t k = 0; k < K; ++k) {
      idx[t * K + k] = (int32_t)top[k].n;
      gate[t * K + k] = std::exp((top[k].hi - k1) + top[k].lo) / den;
      score[t * K + k] = top[k].hi + top[k].lo - lr - lc;
      key_hi[t * K + k] = top[k].hi;
      key_lo[t * K + k] = top[k].lo;
    }
    if ((int64_t)top.size() > K)
      gap[t] = (top[K - 1].hi - top[K].hi) + (top[K - 1].lo - top[K].lo);
    else
      gap[t] = INFINITY;
  });
}

// O6-O7 Expert-Centric Scheduling: tasks t in token-major
// order (Eq.Tasks) carry (token[t], ids[t], gate[t]); tasks whose
// expert lies outside the local range [n_begin, n_end) are not part of this
// plan.  E_active = the distinct in-range experts sorted by id; the
// tau-th of them belongs to group q = floor(tau / B); tasks are
// sorted by (q, token) (Eq.Sort) with a stable counting sort on
// q over the token-major list (tokens then ascend inside each group; tasks of
// one token in one group keep their task order).  With tpb > 0 the batch is
// scheduled in blocks of tpb consecutive tasks (the paper's
// sort applied to each token block in turn): the key is (t / tpb, q).
// Outputs, for local expert
// e = id - n_begin:
//   offsets[e] .. offsets[e+1]   count prefix of expert e (its B = 1 segment)
//   sorted_token/gate/expert     tasks in (q, token) order
//   active[0..n_active)          E_active (local ids, ascending)
//   run_offsets[0..n_runs)       first task of each maximal (q, token) run
void oracle_schedule(int64_t M, const int32_t* ids, const double* gates, const int32_t* tokens,
                     int64_t n_begin, int64_t n_end, int64_t B, int64_t tpb, int32_t* offsets,
                     int32_t* sorted_token, double* sorted_gate, int32_t* sorted_expert,
                     int32_t* active, int64_t* n_active, int32_t* run_offsets, int64_t* n_runs) {
  int64_t n_loc = n_end - n_begin;
  std::vector<int64_t> cnt(n_loc + 1, 0);
  for (int64_t t = 0; t < M; ++t)
    if (ids[t] >= n_begin && ids[t] < n_end) cnt[ids[t] - n_begin + 1]++;
  for (int64_t e = 0; e < n_loc; ++e) cnt[e + 1] += cnt[e];
  for (int64_t e = 0; e <= n_loc; ++e) offsets[e] = (int32_t)cnt[e];
  // E_active and the group of each active expert
  std::vector<int64_t> group(n_loc, -1);
  int64_t na = 0;
  for (int64_t e = 0; e < n_loc; ++e)
    if (offsets[e + 1] > offsets[e]) {
      group[e] = na / B;
      active[na++] = (int32_t)e;
    }
  *n_active = na;
  const int64_t n_groups = (na + B - 1) / B;
  const int64_t n_blocks = tpb > 0 ? (M + tpb - 1) / tpb : 1;
  auto key = [&](int64_t t) {
    return (tpb > 0 ? t / tpb : 0) * n_groups + group[ids[t] - n_begin];
  };
  // stable counting sort of the in-range tasks by (block, group)
  std::vector<int64_t> gstart(n_blocks * n_groups + 1, 0);
  for (int64_t t = 0; t < M; ++t)
    if (ids[t] >= n_begin && ids[t] < n_end) gstart[key(t) + 1]++;
  for (int64_t q = 0; q < n_blocks * n_groups; ++q) gstart[q + 1] += gstart[q];
  std::vector<int64_t> skey(M);
  for (int64_t t = 0; t < M; ++t) {  // visits tasks in t order: stable
    if (ids[t] < n_begin || ids[t] >= n_end) continue;
    const int64_t e = ids[t] - n_begin;
    const int64_t p = gstart[key(t)]++;
    skey[p] = key(t);
    sorted_token[p] = tokens[t];
    sorted_gate[p] = gates[t];
    sorted_expert[p] = (int32_t)e;
  }
  // runs: maximal stretches of equal (group, token)
  const int64_t m_loc = offsets[n_loc];
  int64_t nr = 0;
  for (int64_t p = 0; p < m_loc; ++p)
    if (p == 0 || sorted_token[p] != sorted_token[p - 1] || skey[p] != skey[p - 1])
      run_offsets[nr++] = (int32_t)p;
  *n_runs = nr;
}

// Eq.Grouped executed run by run: for every run (group q,
// token l) and every task (e, g) in it, y[l] += g * sigma(x_l . W_loc[e]) *
// V_loc[e]; the per-run partial is accumulated first and then scatter-added.
void oracle_routed_grouped(int64_t L, int64_t d, int64_t m_loc, int64_t n_runs,
                           const int32_t* run_offsets, const int32_t* sorted_token,
                           const int32_t* sorted_expert, const double* sorted_gate, const double* x,
                           const double* W_loc, const double* V_loc, int act, double* y) {
  for (int64_t i = 0; i < L * d; ++i) y[i] = 0.0;
  std::vector<double> part(d);
  for (int64_t r = 0; r < n_runs; ++r) {
    const int64_t b = run_offsets[r], e = r + 1 < n_runs ? run_offsets[r + 1] : m_loc;
    const int64_t l = sorted_token[b];
    std::fill(part.begin(), part.end(), 0.0);
    for (int64_t p = b; p < e; ++p) {
      const double* w = W_loc + (int64_t)sorted_expert[p] * d;
      const double* v = V_loc + (int64_t)sorted_expert[p] * d;
      double z = 0.0;
      for (int64_t c = 0; c < d; ++c) z += x[l * d + c] * w[c];
      const double a = sorted_gate[p] * act_fn(z, act);
      for (int64_t c = 0; c < d; ++c) part[c] += a * v[c];
    }
    for (int64_t c = 0; c < d; ++c) y[l * d + c] += part[c];
  }
}

// O8 routed branch, token-centric -- the definition (Eq.Assemble,
// PAPER:182-186; Eq.Atomic): for every token l,
// y[l] = sum_{head,k} g * sigma(x_l . W[n]) * V[n], dot products summed
// sequentially in double.  ids index the (possibly compacted) tables W, V.
void oracle_routed_token_centric(int64_t L, int64_t d, int64_t HK, const double* x,
                                 const double* W, const double* V, const int32_t* ids,
                                 const double* gates, int act, double* y, int nthreads) {
  parallel_for(L, nthreads, [&](int64_t l) {
    double* yl = y + l * d;
    for (int64_t c = 0; c < d; ++c) yl[c] = 0.0;
    for (int64_t k = 0; k < HK; ++k) {
      int64_t n = ids[l * HK + k];
      double z = 0.0;
      for (int64_t c = 0; c < d; ++c) z += x[l * d + c] * W[n * d + c];
      double a = gates[l * HK + k] * act_fn(z, act);
      for (int64_t c = 0; c < d; ++c) yl[c] += a * V[n * d + c];
    }
  });
}

// O9 routed branch, expert-centric (Eq.Grouped, with B = 1 so
// G_q is one-hot): walk the plan expert by expert; each expert's W/V rows are
// used for its whole token group, results scatter-added into y.
void oracle_routed_expert_centric(int64_t L, int64_t d, int64_t n_loc, const int32_t* offsets,
                                  const int32_t* sorted_token, const double* sorted_gate,
                                  const double* x, const double* W_loc, const double* V_loc,
                                  int act, double* y) {
  for (int64_t i = 0; i < L * d; ++i) y[i] = 0.0;
  for (int64_t e = 0; e < n_loc; ++e) {
    const double* w = W_loc + e * d;
    const double* v = V_loc + e * d;
    for (int64_t p = offsets[e]; p < offsets[e + 1]; ++p) {
      int64_t l = sorted_token[p];
      double z = 0.0;
      for (int64_t c = 0; c < d; ++c) z += x[l * d + c] * w[c];
      double a = sorted_gate[p] * act_fn(z, act);
      for (int64_t c = 0; c < d; ++c) y[l * d + c] += a * v[c];
    }
  }
}

// O10 shared dense MLP (form per reading Q2 = SwiGLU
// without biases): u = x W_gate, v = x W_up, H = silu(u) * v (not rounded),
// y = H W_down.  w_gu: [2*d_ff][d] (gate rows then up rows), w_down: [d][d_ff].
void oracle_shared_mlp(int64_t L, int64_t d, int64_t d_ff, const double* x, const double* w_gu,
                       const double* w_down, double* y, int nthreads) {
  parallel_for(L, nthreads, [&](int64_t l) {
    std::vector<double> H(d_ff);
    const double* xl = x + l * d;
    for (int64_t f = 0; f < d_ff; ++f) {
      double u = 0.0, v = 0.0;
      for (int64_t c = 0; c < d; ++c) {
        u += xl[c] * w_gu[f * d + c];
        v += xl[c] * w_gu[(d_ff + f) * d + c];
      }
      H[f] = silu(u) * v;
    }
    for (int64_t c = 0; c < d; ++c) {
      double acc = 0.0;
      for (int64_t f = 0; f < d_ff; ++f) acc += H[f] * w_down[c * d_ff + f];
      y[l * d + c] = acc;
    }
  });
}

// Whole layer for a batch of tokens (Eq.MoE):
// exact logits (Q9) -> product selection -> gates -> token-centric routed
// branch (sum over heads) -> + shared MLP.  Used for the CPU baseline timing
// (bench.py cpu_baseline / --impl reference) and as the layer parity oracle.
// subkeys: [h][N_r+N_c][d]; W, V: [N][d] (full tables, or compact tables when
// id_map != nullptr maps flat id -> table row via a sorted list of
// (id, row) pairs of length n_map).
void oracle_layer(int64_t L, int64_t d, int64_t Nr, int64_t Nc, int64_t K, int64_t h,
                  int64_t d_ff, const double* x, const double* subkeys, const double* W,
                  const double* V, const int64_t* id_map, int64_t n_map, const double* w_gu,
                  const double* w_down, int act, double* y, int32_t* idx_out, double* gate_out,
                  int nthreads) {
  int64_t R = Nr + Nc;
  parallel_for(L, nthreads, [&](int64_t l) {
    const double* xl = x + l * d;
    std::vector<float> lg(R);
    std::vector<double> yl(d, 0.0);
    for (int64_t hh = 0; hh < h; ++hh) {
      for (int64_t r = 0; r < R; ++r) lg[r] = exact_dot_rn32(xl, subkeys + (hh * R + r) * d, d);
      std::vector<Key> top;
      select_product(lg.data(), Nr, lg.data() + Nr, Nc, K, top);
      double k1 = top[0].hi + top[0].lo, den = 0.0;
      for (int64_t k = 0; k < K; ++k) den += std::exp((top[k].hi - k1) + top[k].lo);
      for (int64_t k = 0; k < K; ++k) {
        int64_t n = top[k].n;
        double g = std::exp((top[k].hi - k1) + top[k].lo) / den;
        if (idx_out) idx_out[(l * h + hh) * K + k] = (int32_t)n;
        if (gate_out) gate_out[(l * h + hh) * K + k] = g;
        int64_t row = n;
        if (id_map) {  // binary search the (id,row) map
          int64_t lo = 0, hi = n_map - 1;
          while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (id_map[2 * mid] < n) lo = mid + 1; else hi = mid;
          }
          row = id_map[2 * lo + 1];
        }
        double z = 0.0;
        for (int64_t c = 0; c < d; ++c) z += xl[c] * W[row * d + c];
        double a = g * act_fn(z, act);
        for (int64_t c = 0; c < d; ++c) yl[c] += a * V[row * d + c];
      }
    }
    if (d_ff > 0) {
      std::vector<double> H(d_ff);
      for (int64_t f = 0; f < d_ff; ++f) {
        double u = 0.0, v = 0.0;
        for (int64_t c = 0; c < d; ++c) {
          u += xl[c] * w_gu[f * d + c];
          v += xl[c] * w_gu[(d_ff + f) * d + c];
        }
        H[f] = silu(u) * v;
      }
      for (int64_t c = 0; c < d; ++c) {
        double acc = 0.0;
        for (int64_t f = 0; f < d_ff; ++f) acc += H[f] * w_down[c * d_ff + f];
        yl[c] += acc;
      }
    }
    for (int64_t c = 0; c < d; ++c) y[l * d + c] = yl[c];
  });
}

}  // extern "C"
