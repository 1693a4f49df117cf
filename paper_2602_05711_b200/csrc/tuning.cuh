// Measurement overrides of the library's performance choices (the tools/ sweeps), in
// one place.  A shipping build (the default) compiles every knob to its measured
// default and never reads the environment; a measurement build (-DOMNIMOE_MEASURE,
// `python -m paper_2602_05711_b200.build --measure`) reads them ONCE per process from
// OMNIMOE_* environment variables, each validated against its range (out of range or
// garbage: the default).  No knob changes results beyond floating-point summation
// order; they are read once per process, so a workspace size query and the call that
// uses the workspace always agree.
#pragma once
#include <cstdint>
#include <cstdlib>

namespace omni {

struct Tuning {
  int dense_ratio = 40;         // dense routed executor when K * ratio >= N (dense.cu)
  int token_eta_x100 = 200;     // token-centric executor below eta = this / 100 (expert.cu)
  int v_group_max_tasks = 64;   // pass V: 8 tokens per warp when h*K <= this (expert.cu)
  int group_kernel = -1;        // ROWS grouped executor: -1 by d, 0 TMA-staged, 1 register loads
  int l2_hints = 0;             // TMA grouped executor L2 policy bits
  int w_hint = 1, x_hint = 0;   // pass Z (16-byte path) L2 policies of W and x
  int gemm_mfast = -1;          // tcgen05 GEMM tile order: -1 auto, 0 n-fastest, 1 m-fastest
  int select_cta = 0;           // 1: CTA selection kernel for the layer's routing
  int select_warp_group = 0;    // 1: warp-per-token-head variant of the CTA selection
  int i8_cluster = 1;           // exact router GEMM: CTAs per cluster multicasting the token limbs
  int i8_persist = 1;           // exact router GEMM: persistent kernel
  int route_fused = 1;          // N4: per-half top-k' in the exact-logit GEMM epilogue (small K)
  int v_config = 0;             // pass V (CTAs per SM, window) variant, measurement build only
  int64_t ws_pad_counters = 0;  // bytes (<= 16 MB) padded before the layer's work counters
};

inline const Tuning& tuning() {
  static const Tuning t = [] {
    Tuning x;
#ifdef OMNIMOE_MEASURE
    auto get = [](const char* name, long long lo, long long hi, long long dflt) -> long long {
      const char* v = std::getenv(name);
      if (!v || !*v) return dflt;
      char* end = nullptr;
      const long long r = std::strtoll(v, &end, 10);
      return (*end || r < lo || r > hi) ? dflt : r;
    };
    x.dense_ratio = (int)get("OMNIMOE_DENSE_RATIO", 1, 1 << 20, x.dense_ratio);
    x.token_eta_x100 = (int)get("OMNIMOE_TOKEN_ETA_X100", 0, 1 << 20, x.token_eta_x100);
    x.v_group_max_tasks = (int)get("OMNIMOE_V_GROUP_MAX_TASKS", 0, 1 << 20, x.v_group_max_tasks);
    x.group_kernel = (int)get("OMNIMOE_GROUP_KERNEL", -1, 1, x.group_kernel);
    x.l2_hints = (int)get("OMNIMOE_L2_HINTS", 0, 15, x.l2_hints);
    x.w_hint = (int)get("OMNIMOE_W_HINT", 0, 1, x.w_hint);
    x.x_hint = (int)get("OMNIMOE_X_HINT", 0, 1, x.x_hint);
    x.gemm_mfast = (int)get("OMNIMOE_GEMM_MFAST", -1, 1, x.gemm_mfast);
    x.select_cta = (int)get("OMNIMOE_SELECT_CTA", 0, 1, x.select_cta);
    x.select_warp_group = (int)get("OMNIMOE_SELECT_WARP_GROUP", 0, 1, x.select_warp_group);
    x.i8_cluster = (int)get("OMNIMOE_I8_CLUSTER", 1, 4, x.i8_cluster);
    x.i8_persist = (int)get("OMNIMOE_I8_PERSIST", 0, 1, x.i8_persist);
    x.route_fused = (int)get("OMNIMOE_ROUTE_FUSED", 0, 1, x.route_fused);
    x.v_config = (int)get("OMNIMOE_V_CONFIG", 0, 6, x.v_config);
    x.ws_pad_counters = get("OMNIMOE_WS_PAD_COUNTERS", 0, 16ll << 20, x.ws_pad_counters);
#endif
    return x;
  }();
  return t;
}

}  // namespace omni
