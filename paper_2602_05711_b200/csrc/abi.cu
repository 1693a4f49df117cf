// C ABI of libomnimoe (include/omnimoe.h): argument validation, workspace
// carving, and the per-call kernel sequence.  No device allocation, no host
// synchronisation, no CPU fallback.
#include <mutex>
#include <string>
#include <map>
#include <set>
#include <tuple>
#include <vector>

#include "backward.cuh"
#include "ep.cuh"
#include "gemm.cuh"
#include "router.cuh"
#include "schedule.cuh"

namespace omni {

namespace {
thread_local std::string g_err;
thread_local int g_launches = 0;
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int n) { g_launches += n; }
void reset_launch_count() { g_launches = 0; }

namespace {
// per-device facts, queried once per device under a lock
struct DeviceInfo {
  int major = 0, minor = 0, sms = 0;
};
std::mutex g_dev_mu;
std::map<int, DeviceInfo> g_dev;
// (kernel, device) -> the largest dynamic shared memory size applied so far: the attribute
// only ever rises, so every smaller launch stays valid
std::map<std::pair<const void*, int>, int> g_smem_attr;

int current_device() {
  int dev = 0;
  return cudaGetDevice(&dev) == cudaSuccess ? dev : -1;
}
DeviceInfo device_info(int dev) {
  std::lock_guard<std::mutex> g(g_dev_mu);
  auto it = g_dev.find(dev);
  if (it != g_dev.end()) return it->second;
  DeviceInfo di;
  cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&di.minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
  g_dev[dev] = di;
  return di;
}
}  // namespace

int num_sms() {
  const int dev = current_device();
  const int n = dev < 0 ? 0 : device_info(dev).sms;
  return n > 0 ? n : 148;
}

bool set_smem_attr(const void* func, int bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_dev_mu);
  auto it = g_smem_attr.find(std::make_pair(func, dev));
  if (it != g_smem_attr.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  g_smem_attr[std::make_pair(func, dev)] = bytes;
  return true;
}

namespace {

omnimoe_status check_device() {
  const int dev = current_device();
  if (dev < 0) {
    set_error("no CUDA device");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  const DeviceInfo di = device_info(dev);
  if (!(di.major == 10 && di.minor == 0)) {
    set_error("device " + std::to_string(dev) + " is sm_" + std::to_string(di.major) + std::to_string(di.minor) +
              "; libomnimoe is built for sm_100a only");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  return OMNIMOE_OK;
}

std::string dims_str(const omnimoe_dims& d) {
  return "(d=" + std::to_string(d.d) + ", n_rows=" + std::to_string(d.n_rows) +
         ", n_cols=" + std::to_string(d.n_cols) + ", K=" + std::to_string(d.top_k) +
         ", h=" + std::to_string(d.n_heads) + ", d_ff=" + std::to_string(d.d_ff) + ")";
}

omnimoe_status validate_dims(const omnimoe_dims* dp) {
  if (!dp) {
    set_error("dims is null");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  const omnimoe_dims& d = *dp;
  if (d.d < 8 || d.d % 8 != 0 || d.n_rows < 1 || d.n_cols < 1 || d.top_k < 1 || d.n_heads < 1 ||
      d.d_ff < 0 || (d.d_ff > 0 && d.d_ff % 8 != 0)) {
    set_error("invalid dims " + dims_str(d) + ": need d >= 8, d % 8 == 0, N_r, N_c, K, h >= 1, d_ff % 8 == 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (d.dtype != OMNIMOE_BF16 && d.dtype != OMNIMOE_F32) {
    set_error("unknown dtype " + std::to_string(d.dtype));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (d.act != OMNIMOE_SILU && d.act != OMNIMOE_IDENTITY) {
    set_error("unknown activation " + std::to_string(d.act));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (d.router == OMNIMOE_ROUTER_DENSE && d.dtype != OMNIMOE_BF16) {
    set_error("the dense-router ablation runs in bf16 only");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (d.router != OMNIMOE_ROUTER_EXACT && d.router != OMNIMOE_ROUTER_EXACT_F64 && d.router != OMNIMOE_ROUTER_DENSE) {
    set_error("unknown router mode " + std::to_string(d.router));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (d.group_size < 0 || d.token_blocks < 0) {
    set_error("group_size and token_blocks must be >= 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (d.v_band_bytes < 0 || (d.flags & ~(int64_t)OMNIMOE_FLAG_ACT_BF16) != 0) {
    set_error("v_band_bytes must be >= 0 and flags a set of OMNIMOE_FLAG_* " + dims_str(d));
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (d.route_order != OMNIMOE_ORDER_KEY && d.route_order != OMNIMOE_ORDER_CANDIDATE) {
    set_error("unknown route order " + std::to_string(d.route_order));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (d.v_layout != OMNIMOE_V_ROWS && d.v_layout != OMNIMOE_V_SLICED) {
    set_error("unknown V layout " + std::to_string(d.v_layout));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (d.v_layout == OMNIMOE_V_SLICED) {
    if (d.dtype != OMNIMOE_BF16 || d.d % 64 != 0 || d.d > 2048) {
      set_error("V_SLICED layout: bf16 with d % 64 == 0 and d <= 2048 " + dims_str(d));
      return OMNIMOE_ERR_UNSUPPORTED;
    }
    if (d.expert_kernel != OMNIMOE_EXPERT_AUTO && d.expert_kernel != OMNIMOE_EXPERT_SLICED) {
      set_error("V_SLICED layout runs the SLICED executor only (expert_kernel AUTO or SLICED)");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
  } else if (d.expert_kernel == OMNIMOE_EXPERT_SLICED) {
    set_error("expert kernel SLICED needs dims.v_layout == OMNIMOE_V_SLICED");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (d.expert_kernel < OMNIMOE_EXPERT_AUTO || d.expert_kernel > OMNIMOE_EXPERT_SLICED) {
    set_error("unknown expert kernel " + std::to_string(d.expert_kernel));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  {
    const int64_t B = resolve_group_size(d);
    if ((d.expert_kernel == OMNIMOE_EXPERT_WARP && B != 1) || (d.expert_kernel == OMNIMOE_EXPERT_GROUP && B < 2)) {
      set_error("expert kernel " + std::to_string(d.expert_kernel) + " does not match group size B=" +
                std::to_string(B) + " (WARP needs B = 1, GROUP needs B > 1)");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
  }
  const int64_t N = d.n_rows * d.n_cols;
  if (d.top_k > N) {
    set_error("K=" + std::to_string(d.top_k) + " exceeds N=" + std::to_string(N) + " " + dims_str(d));
    return OMNIMOE_ERR_SHAPE;
  }
  if (N >= (int64_t(1) << 31) - 1) {
    set_error("N=" + std::to_string(N) + " must be < 2^31 - 1 (int32 expert ids)");
    return OMNIMOE_ERR_SHAPE;
  }
  return OMNIMOE_OK;
}

// the int8 limb GEMM is exact while every int32 partial sum fits: |digit products| <= 2^14 summed
// over d terms, so d < 2^16; wider rows take the exact fp64 double-double kernel
bool i8_logits(const omnimoe_dims& d) {
  return d.dtype == OMNIMOE_BF16 && d.router == OMNIMOE_ROUTER_EXACT && d.d < 65536;
}

bool dense_router(const omnimoe_dims& d) { return d.router == OMNIMOE_ROUTER_DENSE; }
// logits per token-head: N_r + N_c (Cartesian) or N (dense ablation)
int64_t logit_cols(const omnimoe_dims& d) { return dense_router(d) ? d.n_rows * d.n_cols : d.n_rows + d.n_cols; }

size_t route_ws(const omnimoe_dims& d, int64_t L, void* ws, float** logits, void** sub_ws,
                uint32_t** cand = nullptr, bool with_cand = true, void** fused_ws = nullptr) {
  Carver c(ws);
  const int64_t T = L * d.n_heads;
  float* lg = c.take<float>((size_t)std::max<int64_t>(T, 1) * logit_cols(d));
  void* sw = c.take<char>(dense_router(d) ? 0 : exact_logits_ws_bytes(d, L));
  uint32_t* ct = c.take<uint32_t>(dense_router(d) || !with_cand ? 0 : select_cand_ws_bytes(d) / 4);
  // N4 (small K): the epilogue's per-half lists; zero bytes where the fused path does not apply
  void* fw = c.take<char>(dense_router(d) ? 0 : fused_route_bytes(d, L));
  if (logits) *logits = lg;
  if (sub_ws) *sub_ws = sw;
  if (cand) *cand = ct;
  if (fused_ws) *fused_ws = fw;
  return c.bytes();
}

size_t elem_size(const omnimoe_dims& d) { return d.dtype == OMNIMOE_BF16 ? 2 : 4; }
// bf16 mode carries the shared MLP's hidden activations H into GEMM-2 as a bf16 pair
// [hi | lo] (~16 significant bits; reading Q16) whenever d_ff is a whole number of 64-wide
// K blocks; otherwise as one bf16 value
bool h_split(const omnimoe_dims& d) { return d.dtype == OMNIMOE_BF16 && d.d_ff % 64 == 0; }
int64_t h_cols(const omnimoe_dims& d) { return std::max<int64_t>(d.d_ff, 1) * (h_split(d) ? 2 : 1); }
size_t h_bytes(const omnimoe_dims& d, int64_t L) { return (size_t)L * h_cols(d) * elem_size(d); }

struct LayerWs {
  void* route_ws;
  size_t route_bytes;
  int32_t* idx;
  float* gate;
  omnimoe_plan plan;
  void* sched_ws;
  float* y_routed;
  void* H;
  void* expert_ws;
  uint32_t* cand;
};

size_t layer_ws(const omnimoe_dims& d, int64_t L, void* ws, LayerWs* o) {
  Carver c(ws);
  const int64_t N = d.n_rows * d.n_cols;
  const int64_t M = L * d.n_heads * d.top_k;
  // the selection's candidate table is carved last, so that the other offsets do not
  // depend on it: the SLICED pass V is sensitive to where the plan arrays fall (C5: 55.0
  // ms with this layout, 58.7-59.2 ms with everything after the route scratch shifted by
  // 14 KB, 64 KB or 1 MB -- DESIGN.md §10)
  const size_t rb = route_ws(d, L, nullptr, nullptr, nullptr, nullptr, false);
  void* rw = c.take<char>(rb);
  int32_t* idx = c.take<int32_t>((size_t)std::max<int64_t>(M, 1));
  float* gate = c.take<float>((size_t)std::max<int64_t>(M, 1));
  int32_t* off = c.take<int32_t>(N + 1);
  int32_t* st = c.take<int32_t>((size_t)std::max<int64_t>(M, 1));
  float* sg = c.take<float>((size_t)std::max<int64_t>(M, 1));
  int32_t* act = c.take<int32_t>(N);
  int32_t* na = c.take<int32_t>(1);
  int32_t* se = c.take<int32_t>((size_t)std::max<int64_t>(M, 1));
  int32_t* ro = c.take<int32_t>((size_t)M + 1);
  int32_t* nr = c.take<int32_t>(1);
  const bool sliced = d.v_layout == OMNIMOE_V_SLICED;
  int32_t* stask = sliced ? c.take<int32_t>((size_t)std::max<int64_t>(M, 1)) : nullptr;
  int32_t* tpair = sliced ? c.take<int32_t>(2 * (size_t)std::max<int64_t>(M, 1)) : nullptr;
  int32_t* toff = sliced ? c.take<int32_t>((size_t)L * (resolve_v_bands(d, N, L) + 1) + 1) : nullptr;
  const size_t sb = schedule_ws_bytes(M, N);
  void* sw = c.take<char>(sb);
  float* yr = c.take<float>((size_t)L * d.d);
  // measurement override: pad before the executor's work counters (placement study)
  if (tuning().ws_pad_counters) c.take<char>((size_t)tuning().ws_pad_counters);
  void* ew = c.take<char>(layer_uses_dense_executor(d, L) ? dense_expert_ws_bytes(d, L) : expert_ws_bytes(d, L));
  void* H = c.take<char>(h_bytes(d, L));
  uint32_t* cand = c.take<uint32_t>(dense_router(d) ? 0 : select_cand_ws_bytes(d) / 4);
  if (o) {
    o->cand = cand;
    o->route_ws = rw;
    o->route_bytes = rb;
    o->idx = idx;
    o->gate = gate;
    o->plan = omnimoe_plan{off, st, sg, act, na, 0, N, se, ro, nr, stask, tpair, toff, L};
    o->sched_ws = sw;
    o->y_routed = yr;
    o->expert_ws = ew;
    o->H = H;
  }
  return c.bytes();
}

omnimoe_status check_ws(size_t have, size_t need, const char* who) {
  if (have < need) {
    set_error(std::string(who) + ": workspace of " + std::to_string(have) + " bytes < required " +
              std::to_string(need));
    return OMNIMOE_ERR_WORKSPACE;
  }
  return OMNIMOE_OK;
}

omnimoe_status logits_impl(const omnimoe_dims& d, int64_t L, const void* x, const void* subkeys, float* logits,
                           void* sub_ws, cudaStream_t st) {
  const int NC = (int)(d.n_heads * (d.n_rows + d.n_cols));
  if (dense_router(d)) {  // ablation: the dense projection on the bf16 GEMM engine
    GemmArgs ga;
    ga.M = (int)L;
    ga.N = (int)(d.n_heads * d.n_rows * d.n_cols);
    ga.K = (int)d.d;
    ga.out_f32 = logits;
    return gemm_bf16(EPI_F32, x, subkeys, ga, st);
  }
  if (i8_logits(d)) return exact_logits(d, L, x, subkeys, logits, sub_ws, st);
  return launch_exact_dd(d.dtype, x, subkeys, (int)d.d, NC, (int)L, logits, 0, nullptr, nullptr, st);
}

// a1 (exact logits, Q9) -> a2 + a3 (select_kernel)
omnimoe_status route_impl(const omnimoe_dims& d, int64_t L, const void* x, const void* subkeys,
                          int32_t* idx, float* gate, float* score, void* ws, cudaStream_t st, int sorted = 1,
                          uint32_t* cand_ws = nullptr) {
  float* logits;
  void* sub_ws;
  void* fused_ws = nullptr;
  uint32_t* cand = cand_ws;
  route_ws(d, L, ws, &logits, &sub_ws, cand_ws ? nullptr : &cand, cand_ws == nullptr, &fused_ws);
  if (dense_router(d)) {
    OMNI_TRY(logits_impl(d, L, x, subkeys, logits, sub_ws, st));
    return launch_dense_select(d, L * d.n_heads, logits, idx, gate, score, st);
  }
  SelectParams sp;
  size_t smem;
  OMNI_TRY(select_params(d, L * d.n_heads, &sp, &smem));
  sp.sorted = sorted;
  if (i8_logits(d) && fused_kp(d, L) > 0) {  // N4: per-half top-k' in the GEMM epilogue
    FusedRoute fr;
    OMNI_TRY(exact_logits_fused(d, L, x, subkeys, logits, sub_ws, fused_ws, score != nullptr, &fr, st));
    return launch_select(sp, smem, logits, idx, gate, score, cand, st, &fr);
  }
  OMNI_TRY(logits_impl(d, L, x, subkeys, logits, sub_ws, st));
  return launch_select(sp, smem, logits, idx, gate, score, cand, st);
}

// shared MLP GEMM-1: H = SiLU(x W_gate^T) * (x W_up^T) (the bf16 pair [hi | lo] when split)
omnimoe_status mlp_hidden(const omnimoe_dims& d, int64_t L, const void* x, const void* wgu, void* H,
                          cudaStream_t st) {
  GemmArgs g1;
  g1.M = (int)L;
  g1.N = (int)d.d_ff;
  g1.K = (int)d.d;
  g1.out = H;
  g1.h_split = h_split(d);
  if (d.dtype == OMNIMOE_BF16) return gemm_bf16(EPI_SWIGLU, x, wgu, g1, st);
  return gemm_f32(EPI_SWIGLU, static_cast<const float*>(x), static_cast<const float*>(wgu), g1, st);
}
// shared MLP GEMM-2 + combine: y = H W_down^T + y_routed
omnimoe_status mlp_out(const omnimoe_dims& d, int64_t L, const void* H, const void* wdown, const float* y_routed,
                       void* y, cudaStream_t st) {
  GemmArgs g2;
  g2.M = (int)L;
  g2.N = (int)d.d;
  g2.K = (int)h_cols(d);  // y = [H_hi | H_lo] [W_down | W_down]^T when split
  g2.b_kwrap = h_split(d) ? (int)d.d_ff : 0;
  g2.out = y;
  g2.addend = y_routed;
  if (d.dtype == OMNIMOE_BF16) return gemm_bf16(EPI_ADD, H, wdown, g2, st);
  return gemm_f32(EPI_ADD, static_cast<const float*>(H), static_cast<const float*>(wdown), g2, st);
}
omnimoe_status mlp_impl(const omnimoe_dims& d, int64_t L, const void* x, const void* wgu,
                        const void* wdown, const float* y_routed, void* y, void* H, cudaStream_t st) {
  OMNI_TRY(mlp_hidden(d, L, x, wgu, H, st));
  return mlp_out(d, L, H, wdown, y_routed, y, st);
}

__global__ void cast_out_kernel(const float* __restrict__ in, void* __restrict__ out, int64_t n, int bf16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (bf16) reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(in[i]);
    else reinterpret_cast<float*>(out)[i] = in[i];
  }
}

#define OMNI_NONNULL(p, name)                                  \
  do {                                                         \
    if (!(p)) {                                                \
      set_error(std::string(name) + " must not be null");      \
      return OMNIMOE_ERR_INVALID_ARGUMENT;                     \
    }                                                          \
  } while (0)

}  // namespace
}  // namespace omni

using namespace omni;

extern "C" {

omnimoe_status omnimoe_workspace_size(const omnimoe_dims* dims, int64_t L, int which, size_t* bytes) {
  OMNI_TRY(validate_dims(dims));
  OMNI_NONNULL(bytes, "bytes");
  if (L < 0) {
    set_error("L must be >= 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  const omnimoe_dims& d = *dims;
  switch (which) {
    case OMNIMOE_WS_ROUTE: *bytes = route_ws(d, L, nullptr, nullptr, nullptr); break;
    case OMNIMOE_WS_SCHEDULE: *bytes = schedule_ws_bytes(L, d.n_rows * d.n_cols); break;
    case OMNIMOE_WS_EXPERT: *bytes = expert_ws_bytes(d, L); break;
    case OMNIMOE_WS_LAYER: *bytes = layer_ws(d, L, nullptr, nullptr); break;
    case OMNIMOE_WS_ROUTER_BWD: *bytes = router_bwd_ws_bytes(d, L); break;
    case OMNIMOE_WS_MLP_BWD: *bytes = mlp_bwd_ws_bytes(d, L); break;
    case OMNIMOE_WS_MLP: *bytes = h_bytes(d, L); break;
    case OMNIMOE_WS_EXPERT_BWD: *bytes = expert_bwd_ws_bytes(d, L); break;
    default:
      set_error("unknown workspace selector " + std::to_string(which));
      return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_route(const omnimoe_dims* dims, int64_t L, const void* x, const void* subkeys,
                             int32_t* idx, float* gate, float* score, void* ws, size_t ws_bytes,
                             omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (L < 0 || L >= (int64_t(1) << 31) / std::max<int64_t>(dims->n_heads * dims->top_k, 1)) {
    set_error("L out of range");
    return OMNIMOE_ERR_SHAPE;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(x, "x");
  OMNI_NONNULL(subkeys, "subkeys");
  OMNI_NONNULL(idx, "idx");
  OMNI_NONNULL(gate, "gate");
  OMNI_NONNULL(ws, "ws");
  OMNI_TRY(check_ws(ws_bytes, route_ws(*dims, L, nullptr, nullptr, nullptr), "route"));
  if (!dense_router(*dims)) {
    SelectParams sp;
    size_t smem;
    OMNI_TRY(select_params(*dims, L * dims->n_heads, &sp, &smem));
  }
  OMNI_TRY(check_device());
  return route_impl(*dims, L, x, subkeys, idx, gate, score, ws, (cudaStream_t)stream,
                    dims->route_order == OMNIMOE_ORDER_CANDIDATE ? 0 : 1);
}

omnimoe_status omnimoe_schedule(const omnimoe_dims* dims, int64_t M, const int32_t* idx, const float* gate,
                                const int32_t* token, const omnimoe_plan* plan, void* ws, size_t ws_bytes,
                                omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  OMNI_NONNULL(plan, "plan");
  const int64_t N = dims->n_rows * dims->n_cols;
  if (plan->expert_begin < 0 || plan->expert_end > N || plan->expert_begin >= plan->expert_end) {
    set_error("plan expert range [" + std::to_string(plan->expert_begin) + ", " +
              std::to_string(plan->expert_end) + ") outside [0, " + std::to_string(N) + ")");
    return OMNIMOE_ERR_SHAPE;
  }
  if (M < 0 || M >= (int64_t(1) << 31) - 1) {
    set_error("M=" + std::to_string(M) + " must be in [0, 2^31-1)");
    return OMNIMOE_ERR_SHAPE;
  }
  OMNI_NONNULL(plan->expert_offsets, "plan.expert_offsets");
  OMNI_NONNULL(plan->active, "plan.active");
  OMNI_NONNULL(plan->n_active, "plan.n_active");
  const int64_t B = resolve_group_size(*dims);
  if (M > 0) {
    OMNI_NONNULL(idx, "idx");
    OMNI_NONNULL(gate, "gate");
    OMNI_NONNULL(plan->sorted_token, "plan.sorted_token");
    OMNI_NONNULL(plan->sorted_gate, "plan.sorted_gate");
    OMNI_NONNULL(plan->sorted_expert, "plan.sorted_expert");
  }
  if (B > 1) {
    OMNI_NONNULL(plan->run_offsets, "plan.run_offsets (group size > 1)");
    OMNI_NONNULL(plan->n_runs, "plan.n_runs (group size > 1)");
  }
  OMNI_NONNULL(ws, "ws");
  const int64_t n_loc = plan->expert_end - plan->expert_begin;
  OMNI_TRY(check_ws(ws_bytes, schedule_ws_bytes(M, n_loc), "schedule"));
  OMNI_TRY(check_device());
  const int64_t hk = dims->n_heads * dims->top_k;
  const int64_t n_tok = plan->n_tokens > 0 ? plan->n_tokens : (M + hk - 1) / hk;
  return schedule_run(M, idx, gate, token, hk, *plan, B, resolve_token_blocks(*dims, (M + hk - 1) / hk),
                      resolve_v_bands(*dims, n_loc, std::max<int64_t>(n_tok, 1)), ws, (cudaStream_t)stream);
}

}  // extern "C"

namespace omni {
namespace {
omnimoe_status expert_fwd_impl(const omnimoe_dims* dims, int64_t L, const void* x, const void* W_loc,
                               const void* V_loc, const omnimoe_plan* plan, float* y_routed, int accumulate,
                               void* ws, size_t ws_bytes, omnimoe_stream_t stream, int passes) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (L < 0) {
    set_error("L must be >= 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(plan, "plan");
  OMNI_NONNULL(x, "x");
  OMNI_NONNULL(W_loc, "W_loc");
  OMNI_NONNULL(V_loc, "V_loc");
  OMNI_NONNULL(y_routed, "y_routed");
  OMNI_NONNULL(plan->expert_offsets, "plan.expert_offsets");
  OMNI_NONNULL(plan->active, "plan.active");
  OMNI_NONNULL(plan->n_active, "plan.n_active");
  OMNI_NONNULL(plan->sorted_token, "plan.sorted_token");
  OMNI_NONNULL(plan->sorted_gate, "plan.sorted_gate");
  OMNI_NONNULL(ws, "ws");
  if (dims->expert_kernel == OMNIMOE_EXPERT_TOKEN) {
    set_error("expert_fwd: OMNIMOE_EXPERT_TOKEN runs from the routing decision (omnimoe_layer_fwd), not a plan");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (resolve_group_size(*dims) > 1) {
    OMNI_NONNULL(plan->sorted_expert, "plan.sorted_expert");
    OMNI_NONNULL(plan->run_offsets, "plan.run_offsets (group size > 1)");
    OMNI_NONNULL(plan->n_runs, "plan.n_runs (group size > 1)");
  }
  if (dims->v_layout == OMNIMOE_V_SLICED) {
    OMNI_NONNULL(plan->sorted_task, "plan.sorted_task (SLICED executor)");
    OMNI_NONNULL(plan->task_pair, "plan.task_pair (SLICED executor)");
    OMNI_NONNULL(plan->token_offsets, "plan.token_offsets (SLICED executor)");
  }
  OMNI_TRY(check_ws(ws_bytes, expert_ws_bytes(*dims, L), "expert_fwd"));
  OMNI_TRY(check_device());
  if (passes != 3) {
    if (dims->v_layout != OMNIMOE_V_SLICED || passes < 1 || passes > 3) {
      set_error("expert_fwd_pass: pass 1 (Z) or 2 (V) of the SLICED executor only");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
    // the measurement entry point times the passes as omnimoe_layer_fwd runs them
    return expert_sliced_run(*dims, L, x, W_loc, V_loc, *plan, y_routed, accumulate, ws, (cudaStream_t)stream,
                             passes, /*act_bf16=*/1);
  }
  return expert_run(*dims, L, x, W_loc, V_loc, *plan, y_routed, accumulate, ws, (cudaStream_t)stream,
                    (dims->flags & OMNIMOE_FLAG_ACT_BF16) ? 1 : 0);
}
}  // namespace
}  // namespace omni

extern "C" {
omnimoe_status omnimoe_expert_fwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* W_loc,
                                  const void* V_loc, const omnimoe_plan* plan, float* y_routed,
                                  int accumulate, void* ws, size_t ws_bytes, omnimoe_stream_t stream) {
  return expert_fwd_impl(dims, L, x, W_loc, V_loc, plan, y_routed, accumulate, ws, ws_bytes, stream, 3);
}

omnimoe_status omnimoe_expert_fwd_pass(const omnimoe_dims* dims, int64_t L, const void* x, const void* W_loc,
                                       const void* V_loc, const omnimoe_plan* plan, float* y_routed,
                                       int accumulate, int pass, void* ws, size_t ws_bytes,
                                       omnimoe_stream_t stream) {
  return expert_fwd_impl(dims, L, x, W_loc, V_loc, plan, y_routed, accumulate, ws, ws_bytes, stream, pass);
}

omnimoe_status omnimoe_shared_mlp(const omnimoe_dims* dims, int64_t L, const void* x, const void* w_gate_up,
                                  const void* w_down, const float* y_routed, void* y, void* ws,
                                  size_t ws_bytes, omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (dims->d_ff < 1) {
    set_error("shared_mlp needs d_ff >= 1");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(x, "x");
  OMNI_NONNULL(w_gate_up, "w_gate_up");
  OMNI_NONNULL(w_down, "w_down");
  OMNI_NONNULL(y, "y");
  OMNI_NONNULL(ws, "ws");
  const size_t need = h_bytes(*dims, L);
  OMNI_TRY(check_ws(ws_bytes, need, "shared_mlp"));
  OMNI_TRY(check_device());
  return mlp_impl(*dims, L, x, w_gate_up, w_down, y_routed, y, ws, (cudaStream_t)stream);
}

omnimoe_status omnimoe_shared_mlp_hidden(const omnimoe_dims* dims, int64_t L, const void* x, const void* w_gate_up,
                                         void* H, size_t H_bytes, omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (dims->d_ff < 1) {
    set_error("shared_mlp_hidden needs d_ff >= 1");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(x, "x");
  OMNI_NONNULL(w_gate_up, "w_gate_up");
  OMNI_NONNULL(H, "H");
  OMNI_TRY(check_ws(H_bytes, h_bytes(*dims, L), "shared_mlp_hidden (H)"));
  OMNI_TRY(check_device());
  return mlp_hidden(*dims, L, x, w_gate_up, H, (cudaStream_t)stream);
}

omnimoe_status omnimoe_shared_mlp_out(const omnimoe_dims* dims, int64_t L, const void* H, size_t H_bytes,
                                      const void* w_down, const float* y_routed, void* y, omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (dims->d_ff < 1) {
    set_error("shared_mlp_out needs d_ff >= 1");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(H, "H");
  OMNI_NONNULL(w_down, "w_down");
  OMNI_NONNULL(y, "y");
  OMNI_TRY(check_ws(H_bytes, h_bytes(*dims, L), "shared_mlp_out (H)"));
  OMNI_TRY(check_device());
  return mlp_out(*dims, L, H, w_down, y_routed, y, (cudaStream_t)stream);
}

omnimoe_status omnimoe_layer_fwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* subkeys,
                                 const void* W, const void* V, const void* w_gate_up, const void* w_down,
                                 void* y, int32_t* idx_out, float* gate_out, void* ws, size_t ws_bytes,
                                 omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  const omnimoe_dims& d = *dims;
  if (L < 0 || L * d.n_heads * d.top_k >= (int64_t(1) << 31) - 1) {
    set_error("L*h*K must be < 2^31-1");
    return OMNIMOE_ERR_SHAPE;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(x, "x");
  OMNI_NONNULL(subkeys, "subkeys");
  OMNI_NONNULL(W, "W");
  OMNI_NONNULL(V, "V");
  OMNI_NONNULL(y, "y");
  OMNI_NONNULL(ws, "ws");
  if (d.d_ff > 0) {
    OMNI_NONNULL(w_gate_up, "w_gate_up");
    OMNI_NONNULL(w_down, "w_down");
  }
  OMNI_TRY(check_ws(ws_bytes, layer_ws(d, L, nullptr, nullptr), "layer_fwd"));
  OMNI_TRY(check_device());
  cudaStream_t st = (cudaStream_t)stream;
  LayerWs w;
  layer_ws(d, L, ws, &w);
  int32_t* idx = idx_out ? idx_out : w.idx;
  float* gate = gate_out ? gate_out : w.gate;
  const int64_t M = L * d.n_heads * d.top_k;
  // the layer does not need the ids sorted by key (the schedule re-sorts the tasks)
  OMNI_TRY(route_impl(d, L, x, subkeys, idx, gate, nullptr, w.route_ws, st, /*sorted=*/0, w.cand));
  const int r_launch = omnimoe_last_launch_count();
  w.plan.n_tokens = L;
  if (layer_uses_token_executor(d, L)) {  // no expert shared by two tasks (or the "w/o ECS" ablation)
    OMNI_TRY(expert_token_run(d, L, x, W, V, idx, gate, 0, d.n_rows * d.n_cols, w.y_routed, 0, st));
  } else if (layer_uses_dense_executor(d, L)) {  // every expert shared by ~100 tokens: two GEMMs
    OMNI_TRY(dense_expert_run(d, L, x, W, V, idx, gate, w.y_routed, w.expert_ws, st));
  } else {
    OMNI_TRY(schedule_run(M, idx, gate, nullptr, d.n_heads * d.top_k, w.plan, resolve_group_size(d),
                          resolve_token_blocks(d, L), resolve_v_bands(d, d.n_rows * d.n_cols, L), w.sched_ws, st));
    OMNI_TRY(expert_run(d, L, x, W, V, w.plan, w.y_routed, 0, w.expert_ws, st, /*act_bf16=*/1));
  }
  if (d.d_ff > 0) {
    OMNI_TRY(mlp_impl(d, L, x, w_gate_up, w_down, w.y_routed, y, w.H, st));
  } else {
    cast_out_kernel<<<num_sms() * 4, 256, 0, st>>>(w.y_routed, y, L * d.d, d.dtype == OMNIMOE_BF16);
    OMNI_CHECK_LAUNCH("cast_out_kernel");
  }
  (void)r_launch;
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_pack_v(const omnimoe_dims* dims, int64_t n, const void* V, void* V_sliced,
                              omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (dims->dtype != OMNIMOE_BF16 || dims->d % 64 != 0) {
    set_error("pack_v: bf16 with d % 64 == 0 " + dims_str(*dims));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (n < 0 || n >= (int64_t(1) << 31)) {
    set_error("pack_v: n out of range");
    return OMNIMOE_ERR_SHAPE;
  }
  if (n == 0) return OMNIMOE_OK;
  OMNI_NONNULL(V, "V");
  OMNI_NONNULL(V_sliced, "V_sliced");
  if (V == V_sliced) {
    set_error("pack_v: V and V_sliced must not alias");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  OMNI_TRY(check_device());
  return pack_v(n, (int)dims->d, V, V_sliced, (cudaStream_t)stream);
}

omnimoe_status omnimoe_expert_fwd_tokens(const omnimoe_dims* dims, int64_t L, const void* x, const void* W,
                                         const void* V, const int32_t* idx, const float* gate, float* y_routed,
                                         int accumulate, omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (L < 0) {
    set_error("L must be >= 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(x, "x");
  OMNI_NONNULL(W, "W");
  OMNI_NONNULL(V, "V");
  OMNI_NONNULL(idx, "idx");
  OMNI_NONNULL(gate, "gate");
  OMNI_NONNULL(y_routed, "y_routed");
  if (dims->v_layout != OMNIMOE_V_ROWS) {
    set_error("expert_fwd_tokens: V in the ROWS layout");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  OMNI_TRY(check_device());
  return expert_token_run(*dims, L, x, W, V, idx, gate, 0, dims->n_rows * dims->n_cols, y_routed, accumulate,
                          (cudaStream_t)stream);
}

omnimoe_status omnimoe_expert_bwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* W_loc,
                                  const void* V_loc, const void* W_sliced, const omnimoe_plan* plan,
                                  const void* dy, float* dx, float* dW_act, float* dV_act, float* dgate,
                                  int accumulate_dx, void* ws, size_t ws_bytes, omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  const omnimoe_dims& d = *dims;
  if (d.dtype != OMNIMOE_BF16 || d.d % 64 != 0 || d.d > 2048) {
    set_error("expert_bwd: bf16 with d % 64 == 0 and d <= 2048 " + dims_str(d));
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (L < 0) {
    set_error("L must be >= 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (L == 0) return OMNIMOE_OK;
  const void* req[] = {x, W_loc, V_loc, W_sliced, plan, dy, dx, dW_act, dV_act, dgate, ws};
  for (const void* p : req)
    if (!p) {
      set_error("expert_bwd: a required pointer is null");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
  OMNI_NONNULL(plan->sorted_task, "plan.sorted_task");
  OMNI_NONNULL(plan->task_pair, "plan.task_pair");
  OMNI_NONNULL(plan->token_offsets, "plan.token_offsets");
  omnimoe_dims ds = d;
  ds.v_layout = OMNIMOE_V_SLICED;
  if (resolve_group_size(d) != 1 && d.group_size != 1) {
    set_error("expert_bwd: needs the expert-major plan (group_size 1 or the SLICED layout)");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  {  // the backward writes dgate in task order through plan.sorted_task: one band (V order = task order)
    const int64_t n_loc = plan->expert_end - plan->expert_begin;
    const int64_t n_tok = plan->n_tokens > 0 ? plan->n_tokens : L;
    if (resolve_v_bands(ds, n_loc, std::max<int64_t>(n_tok, 1)) != 1) {
      set_error("expert_bwd: the plan must have one V band (dims.v_band_bytes >= 128 * n_loc)");
      return OMNIMOE_ERR_UNSUPPORTED;
    }
  }
  OMNI_TRY(check_ws(ws_bytes, expert_bwd_ws_bytes(d, L), "expert_bwd"));
  OMNI_TRY(check_device());
  return expert_bwd_run(ds, L, x, W_loc, V_loc, W_sliced, *plan, dy, dx, dW_act, dV_act, dgate, accumulate_dx, ws,
                        (cudaStream_t)stream);
}

omnimoe_status omnimoe_router_bwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* subkeys,
                                  const int32_t* idx, const float* gate, const float* dgate, float* dx,
                                  int accumulate_dx, float* dsubkeys, void* ws, size_t ws_bytes,
                                  omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (dims->dtype != OMNIMOE_BF16 || dims->router == OMNIMOE_ROUTER_DENSE) {
    set_error("router_bwd: the bf16 Cartesian router only");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (L <= 0) return L == 0 ? OMNIMOE_OK : OMNIMOE_ERR_INVALID_ARGUMENT;
  const void* req[] = {x, subkeys, idx, gate, dgate, dx, dsubkeys, ws};
  for (const void* p : req)
    if (!p) {
      set_error("router_bwd: a required pointer is null");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
  OMNI_TRY(check_ws(ws_bytes, router_bwd_ws_bytes(*dims, L), "router_bwd"));
  OMNI_TRY(check_device());
  return router_bwd_run(*dims, L, x, subkeys, idx, gate, dgate, dx, accumulate_dx, dsubkeys, ws,
                        (cudaStream_t)stream);
}

omnimoe_status omnimoe_shared_mlp_bwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* w_gate_up,
                                      const void* w_down, const void* dy, float* dx, int accumulate_dx,
                                      float* dw_gate_up, float* dw_down, void* ws, size_t ws_bytes,
                                      omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (dims->dtype != OMNIMOE_BF16 || dims->d_ff < 1) {
    set_error("shared_mlp_bwd: bf16 with d_ff >= 1");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (L <= 0) return L == 0 ? OMNIMOE_OK : OMNIMOE_ERR_INVALID_ARGUMENT;
  const void* req[] = {x, w_gate_up, w_down, dy, dx, dw_gate_up, dw_down, ws};
  for (const void* p : req)
    if (!p) {
      set_error("shared_mlp_bwd: a required pointer is null");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
  OMNI_TRY(check_ws(ws_bytes, mlp_bwd_ws_bytes(*dims, L), "shared_mlp_bwd"));
  OMNI_TRY(check_device());
  return mlp_bwd_run(*dims, L, x, w_gate_up, w_down, dy, dx, accumulate_dx, dw_gate_up, dw_down, ws,
                     (cudaStream_t)stream);
}

size_t omnimoe_dense_workspace_size(const omnimoe_dims* dims, int64_t L) {
  if (validate_dims(dims) != OMNIMOE_OK || L < 0) return 0;
  return dense_expert_ws_bytes(*dims, L);
}

omnimoe_status omnimoe_expert_fwd_dense(const omnimoe_dims* dims, int64_t L, const void* x, const void* W,
                                        const void* V, const int32_t* idx, const float* gate, float* y_routed,
                                        void* ws, size_t ws_bytes, omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (dims->dtype != OMNIMOE_BF16 || dims->n_heads != 1 || dims->v_layout != OMNIMOE_V_ROWS) {
    set_error("expert_fwd_dense: bf16, one head, V in the ROWS layout");
    return OMNIMOE_ERR_UNSUPPORTED;
  }
  if (L <= 0) return L == 0 ? OMNIMOE_OK : OMNIMOE_ERR_INVALID_ARGUMENT;
  const void* req[] = {x, W, V, idx, gate, y_routed, ws};
  for (const void* p : req)
    if (!p) {
      set_error("expert_fwd_dense: a required pointer is null");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
  OMNI_TRY(check_ws(ws_bytes, dense_expert_ws_bytes(*dims, L), "expert_fwd_dense"));
  OMNI_TRY(check_device());
  return dense_expert_run(*dims, L, x, W, V, idx, gate, y_routed, ws, (cudaStream_t)stream);
}

int32_t omnimoe_layer_executor(const omnimoe_dims* dims, int64_t L) {
  if (validate_dims(dims) != OMNIMOE_OK || L < 0) return -1;
  if (layer_uses_token_executor(*dims, L)) return OMNIMOE_EXPERT_TOKEN;
  if (layer_uses_dense_executor(*dims, L)) return OMNIMOE_EXPERT_DENSE;
  if (dims->v_layout == OMNIMOE_V_SLICED) return OMNIMOE_EXPERT_SLICED;
  return resolve_group_size(*dims) > 1 ? OMNIMOE_EXPERT_GROUP : OMNIMOE_EXPERT_WARP;
}

omnimoe_status omnimoe_layer_fwd_host(const omnimoe_dims* dims, int64_t L, const void* x_host, void* x_dev,
                                      const void* subkeys, const void* W, const void* V, const void* w_gate_up,
                                      const void* w_down, void* y_dev, void* y_host, int chunks, void* ws,
                                      size_t ws_bytes, omnimoe_stream_t stream, omnimoe_stream_t copy_stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  const omnimoe_dims& d = *dims;
  if (L < 0 || L * d.n_heads * d.top_k >= (int64_t(1) << 31) - 1) {
    set_error("L*h*K must be < 2^31-1");
    return OMNIMOE_ERR_SHAPE;
  }
  if (L == 0) return OMNIMOE_OK;
  const void* req[] = {x_host, x_dev, subkeys, W, V, y_dev, y_host, ws, copy_stream};
  for (const void* p : req)
    if (!p) {
      set_error("layer_fwd_host: a required pointer / stream is null");
      return OMNIMOE_ERR_INVALID_ARGUMENT;
    }
  if (d.d_ff > 0) {
    OMNI_NONNULL(w_gate_up, "w_gate_up");
    OMNI_NONNULL(w_down, "w_down");
  }
  if (chunks < 1 || chunks > 64) {
    set_error("layer_fwd_host: chunks must be in [1, 64]");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  OMNI_TRY(check_ws(ws_bytes, layer_ws(d, L, nullptr, nullptr), "layer_fwd_host"));
  OMNI_TRY(check_device());
  cudaStream_t st = (cudaStream_t)stream, cs = (cudaStream_t)copy_stream;
  // event pool per (thread, device): events belong to the device current when they were created
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    set_error("layer_fwd_host: cudaGetDevice failed");
    return OMNIMOE_ERR_CUDA;
  }
  thread_local std::map<int, std::vector<cudaEvent_t>> pools;
  std::vector<cudaEvent_t>& evs = pools[dev];
  const size_t need = 2 * (size_t)chunks + 2;
  while (evs.size() < need) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      set_error("layer_fwd_host: cannot create events");
      return OMNIMOE_ERR_CUDA;
    }
    evs.push_back(e);
  }
  LayerWs w;
  layer_ws(d, L, ws, &w);
  const size_t eb = elem_size(d);
  const int64_t hk = d.n_heads * d.top_k, M = L * hk;
  const int64_t Lc = (((L + chunks - 1) / chunks) + 127) / 128 * 128;  // whole 128-row GEMM tiles
  int n_ch = 0;
  // 0. the copy stream starts after everything already enqueued on `stream` (earlier work
  //    may still read x_dev, or the caller's allocator may have just recycled it there)
  if (cudaEventRecord(evs[2 * chunks + 1], st) != cudaSuccess || cudaStreamWaitEvent(cs, evs[2 * chunks + 1], 0) != cudaSuccess) {
    set_error("layer_fwd_host: event failed");
    return OMNIMOE_ERR_CUDA;
  }
  // 1. copy x chunk by chunk (copy stream) while routing the chunks already copied:
  //    routing is per token and batch-independent, so chunked routing is bit-identical
  for (int64_t l0 = 0; l0 < L; l0 += Lc, ++n_ch) {
    const int64_t n = std::min(Lc, L - l0);
    if (cudaMemcpyAsync(static_cast<char*>(x_dev) + l0 * d.d * eb, static_cast<const char*>(x_host) + l0 * d.d * eb,
                        n * d.d * eb, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
        cudaEventRecord(evs[n_ch], cs) != cudaSuccess || cudaStreamWaitEvent(st, evs[n_ch], 0) != cudaSuccess) {
      set_error("layer_fwd_host: host-to-device copy failed");
      return OMNIMOE_ERR_CUDA;
    }
    OMNI_TRY(route_impl(d, n, static_cast<const char*>(x_dev) + l0 * d.d * eb, subkeys, w.idx + l0 * hk,
                        w.gate + l0 * hk, nullptr, w.route_ws, st, /*sorted=*/0, w.cand));
    // the shared MLP's GEMM-1 needs only these rows of x: it runs while the next chunk
    // uploads (host-to-device copies here run at ~28 GB/s: 2.4 ms for C3a's x, longer
    // than the routing they overlap)
    if (d.d_ff > 0)
      OMNI_TRY(mlp_hidden(d, n, static_cast<const char*>(x_dev) + l0 * d.d * eb, w_gate_up,
                          static_cast<char*>(w.H) + l0 * h_cols(d) * eb, st));
  }
  // 2. the routed branch over the whole batch (Expert-Centric Scheduling needs every task)
  w.plan.n_tokens = L;
  if (layer_uses_token_executor(d, L)) {
    OMNI_TRY(expert_token_run(d, L, x_dev, W, V, w.idx, w.gate, 0, d.n_rows * d.n_cols, w.y_routed, 0, st));
  } else if (layer_uses_dense_executor(d, L)) {
    OMNI_TRY(dense_expert_run(d, L, x_dev, W, V, w.idx, w.gate, w.y_routed, w.expert_ws, st));
  } else {
    OMNI_TRY(schedule_run(M, w.idx, w.gate, nullptr, hk, w.plan, resolve_group_size(d), resolve_token_blocks(d, L),
                          resolve_v_bands(d, d.n_rows * d.n_cols, L), w.sched_ws, st));
    OMNI_TRY(expert_run(d, L, x_dev, W, V, w.plan, w.y_routed, 0, w.expert_ws, st, /*act_bf16=*/1));
  }
  // 3. shared MLP GEMM-2 (+ combine) chunk by chunk (GEMM-1 ran per chunk above), each chunk
  //    of y copied back on the copy stream while the next is computed
  int c = 0;
  for (int64_t l0 = 0; l0 < L; l0 += Lc, ++c) {
    const int64_t n = std::min(Lc, L - l0);
    void* yc = static_cast<char*>(y_dev) + l0 * d.d * eb;
    if (d.d_ff > 0) {
      GemmArgs g2;
      g2.M = (int)n;
      g2.N = (int)d.d;
      g2.K = (int)h_cols(d);
      g2.b_kwrap = h_split(d) ? (int)d.d_ff : 0;
      g2.out = yc;
      g2.addend = w.y_routed + l0 * d.d;
      const void* Hc = static_cast<const char*>(w.H) + l0 * h_cols(d) * eb;
      if (d.dtype == OMNIMOE_BF16) OMNI_TRY(gemm_bf16(EPI_ADD, Hc, w_down, g2, st));
      else OMNI_TRY(gemm_f32(EPI_ADD, static_cast<const float*>(Hc), static_cast<const float*>(w_down), g2, st));
    } else {
      cast_out_kernel<<<num_sms() * 4, 256, 0, st>>>(w.y_routed + l0 * d.d, yc, n * d.d, d.dtype == OMNIMOE_BF16);
      OMNI_CHECK_LAUNCH("cast_out_kernel");
    }
    if (cudaEventRecord(evs[n_ch + c], st) != cudaSuccess || cudaStreamWaitEvent(cs, evs[n_ch + c], 0) != cudaSuccess ||
        cudaMemcpyAsync(static_cast<char*>(y_host) + l0 * d.d * eb, yc, n * d.d * eb, cudaMemcpyDeviceToHost, cs) !=
            cudaSuccess) {
      set_error("layer_fwd_host: device-to-host copy failed");
      return OMNIMOE_ERR_CUDA;
    }
  }
  // the call completes on `stream` once y is on the host
  if (cudaEventRecord(evs[2 * chunks], cs) != cudaSuccess || cudaStreamWaitEvent(st, evs[2 * chunks], 0) != cudaSuccess) {
    set_error("layer_fwd_host: event failed");
    return OMNIMOE_ERR_CUDA;
  }
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_router_logits(const omnimoe_dims* dims, int64_t L, const void* x, const void* subkeys,
                                     float* logits, int method, void* ws, size_t ws_bytes,
                                     omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(x, "x");
  OMNI_NONNULL(subkeys, "subkeys");
  OMNI_NONNULL(logits, "logits");
  if (method < 0 || method > 2 || (method == 2 && dims->dtype != OMNIMOE_BF16)) {
    set_error("router_logits: method must be 0 (route path), 1 (exact fp64) or 2 (bf16 tcgen05, bf16 only)");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (method == 0) {
    OMNI_NONNULL(ws, "ws");
    OMNI_TRY(check_ws(ws_bytes, route_ws(*dims, L, nullptr, nullptr, nullptr), "router_logits"));
  }
  OMNI_TRY(check_device());
  const omnimoe_dims& d = *dims;
  cudaStream_t st = (cudaStream_t)stream;
  const int NC = (int)(d.n_heads * (d.n_rows + d.n_cols));
  if (method == 0) {
    void* sub_ws;
    route_ws(d, L, ws, nullptr, &sub_ws);
    return logits_impl(d, L, x, subkeys, logits, sub_ws, st);
  }
  if (method == 1) return launch_exact_dd(d.dtype, x, subkeys, (int)d.d, NC, (int)L, logits, 0, nullptr, nullptr, st);
  GemmArgs ga;
  ga.M = (int)L;
  ga.N = NC;
  ga.K = (int)d.d;
  ga.out_f32 = logits;
  return gemm_bf16(EPI_F32, x, subkeys, ga, st);
}

omnimoe_status omnimoe_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, const void* B, float* C,
                                 omnimoe_stream_t stream) {
  reset_launch_count();
  if (M < 0 || N < 0 || K < 8 || K % 8 != 0 || M >= (int64_t(1) << 31) || N >= (int64_t(1) << 31)) {
    set_error("gemm: need M, N >= 0 and K >= 8 with K % 8 == 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (M == 0 || N == 0) return OMNIMOE_OK;
  OMNI_NONNULL(A, "A");
  OMNI_NONNULL(B, "B");
  OMNI_NONNULL(C, "C");
  OMNI_TRY(check_device());
  GemmArgs ga;
  ga.M = (int)M;
  ga.N = (int)N;
  ga.K = (int)K;
  ga.out_f32 = C;
  return gemm_bf16(EPI_F32, A, B, ga, (cudaStream_t)stream);
}

omnimoe_status omnimoe_ep_pack_workspace_size(int64_t L, int32_t R, size_t* bytes) {
  OMNI_NONNULL(bytes, "bytes");
  if (L < 0 || R < 1 || R > kMaxRanks) {
    set_error("ep: need L >= 0 and 1 <= R <= " + std::to_string(kMaxRanks));
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  *bytes = ep_pack_ws_bytes(L, R);
  return OMNIMOE_OK;
}

omnimoe_status omnimoe_ep_pack(const omnimoe_dims* dims, int64_t L, int32_t R, const void* x, const int32_t* idx,
                               const float* gate, void* x_send, int32_t* rec_send, int32_t* inv, int32_t* offsets,
                               int64_t* counts, void* ws, size_t ws_bytes, omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  const omnimoe_dims& d = *dims;
  const int64_t N = d.n_rows * d.n_cols;
  if (R < 1 || R > kMaxRanks || N % R != 0) {
    set_error("ep_pack: R=" + std::to_string(R) + " must divide N=" + std::to_string(N) + " and be <= " +
              std::to_string(kMaxRanks));
    return OMNIMOE_ERR_SHAPE;
  }
  if (L < 0 || L * d.n_heads * d.top_k >= (int64_t(1) << 31) - 1) {
    set_error("ep_pack: L*h*K out of range");
    return OMNIMOE_ERR_SHAPE;
  }
  OMNI_NONNULL(offsets, "offsets");
  OMNI_NONNULL(ws, "ws");
  if (L > 0) {
    OMNI_NONNULL(x, "x");
    OMNI_NONNULL(idx, "idx");
    OMNI_NONNULL(gate, "gate");
    OMNI_NONNULL(x_send, "x_send");
    OMNI_NONNULL(rec_send, "rec_send");
    OMNI_NONNULL(inv, "inv");
  }
  OMNI_TRY(check_ws(ws_bytes, ep_pack_ws_bytes(L, R), "ep_pack"));
  OMNI_TRY(check_device());
  return ep_pack(d.dtype, L, (int)d.d, (int)(d.n_heads * d.top_k), R, N / R, x, idx, gate, x_send, rec_send, inv,
                 offsets, counts, ws, (cudaStream_t)stream);
}

omnimoe_status omnimoe_ep_unpack(int64_t M, int32_t R, const int32_t* rec, const int64_t* task_off,
                                 const int64_t* tok_off, int32_t* ids, float* gate, int32_t* token,
                                 omnimoe_stream_t stream) {
  reset_launch_count();
  if (M < 0 || R < 1 || R > kMaxRanks) {
    set_error("ep_unpack: need M >= 0 and 1 <= R <= " + std::to_string(kMaxRanks));
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (M == 0) return OMNIMOE_OK;
  OMNI_NONNULL(rec, "rec");
  OMNI_NONNULL(task_off, "task_off");
  OMNI_NONNULL(tok_off, "tok_off");
  OMNI_NONNULL(ids, "ids");
  OMNI_NONNULL(gate, "gate");
  OMNI_NONNULL(token, "token");
  OMNI_TRY(check_device());
  return ep_unpack(rec, M, R, task_off, tok_off, ids, gate, token, (cudaStream_t)stream);
}

omnimoe_status omnimoe_ep_partials(int64_t rows, const omnimoe_dims* dims, const float* y_part, void* y_bf16,
                                   omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (rows < 0 || dims->d % 4 != 0) {
    set_error("ep_partials: rows >= 0 and d % 4 == 0");
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (rows == 0) return OMNIMOE_OK;
  OMNI_NONNULL(y_part, "y_part");
  OMNI_NONNULL(y_bf16, "y_bf16");
  OMNI_TRY(check_device());
  return ep_partials_bf16(y_part, rows * dims->d, y_bf16, (cudaStream_t)stream);
}

omnimoe_status omnimoe_ep_combine(const omnimoe_dims* dims, int64_t L, int32_t R, const void* y_ret,
                                  int32_t y_ret_bf16, const int32_t* inv, const int64_t* tok_off, float* y_routed,
                                  omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_TRY(validate_dims(dims));
  if (L < 0 || R < 1 || R > kMaxRanks) {
    set_error("ep_combine: need L >= 0 and 1 <= R <= " + std::to_string(kMaxRanks));
    return OMNIMOE_ERR_INVALID_ARGUMENT;
  }
  if (L == 0) return OMNIMOE_OK;
  OMNI_NONNULL(inv, "inv");
  OMNI_NONNULL(tok_off, "tok_off");
  OMNI_NONNULL(y_routed, "y_routed");
  OMNI_TRY(check_device());
  return ep_combine(y_ret, y_ret_bf16 != 0, inv, tok_off, L, (int)dims->d, R, y_routed, (cudaStream_t)stream);
}

omnimoe_status omnimoe_load_stats(const omnimoe_plan* plan, double* stats, void* ws, size_t ws_bytes,
                                  omnimoe_stream_t stream) {
  reset_launch_count();
  OMNI_NONNULL(plan, "plan");
  OMNI_NONNULL(plan->expert_offsets, "plan.expert_offsets");
  OMNI_NONNULL(stats, "stats");
  OMNI_NONNULL(ws, "ws");
  if (plan->expert_end <= plan->expert_begin) {
    set_error("load_stats: empty expert range");
    return OMNIMOE_ERR_SHAPE;
  }
  OMNI_TRY(check_ws(ws_bytes, load_stats_ws_bytes(), "load_stats"));
  OMNI_TRY(check_device());
  return load_stats_run(*plan, stats, ws, (cudaStream_t)stream);
}

size_t omnimoe_load_stats_workspace_size(void) { return load_stats_ws_bytes(); }

int omnimoe_last_launch_count(void) { return g_launches; }

int64_t omnimoe_group_size(const omnimoe_dims* dims) {
  if (validate_dims(dims) != OMNIMOE_OK) return 0;
  return resolve_group_size(*dims);
}

int64_t omnimoe_v_bands(const omnimoe_dims* dims, int64_t n_loc, int64_t n_tok) {
  if (validate_dims(dims) != OMNIMOE_OK || n_loc < 1 || n_tok < 1) return 0;
  return resolve_v_bands(*dims, n_loc, n_tok);
}

int64_t omnimoe_token_blocks(const omnimoe_dims* dims, int64_t L) {
  if (validate_dims(dims) != OMNIMOE_OK || L < 0) return 0;
  return resolve_token_blocks(*dims, L);
}

const char* omnimoe_status_string(omnimoe_status s) {
  switch (s) {
    case OMNIMOE_OK: return "OMNIMOE_OK";
    case OMNIMOE_ERR_INVALID_ARGUMENT: return "OMNIMOE_ERR_INVALID_ARGUMENT";
    case OMNIMOE_ERR_SHAPE: return "OMNIMOE_ERR_SHAPE";
    case OMNIMOE_ERR_UNSUPPORTED: return "OMNIMOE_ERR_UNSUPPORTED";
    case OMNIMOE_ERR_WORKSPACE: return "OMNIMOE_ERR_WORKSPACE";
    case OMNIMOE_ERR_CUDA: return "OMNIMOE_ERR_CUDA";
  }
  return "OMNIMOE_UNKNOWN_STATUS";
}

const char* omnimoe_last_error(void) { return g_err.c_str(); }

}  // extern "C"
