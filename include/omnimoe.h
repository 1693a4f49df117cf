/*
 * omnimoe.h -- C ABI of the B200-native OmniMoE atomic-expert layer forward
 * (arXiv 2602.05711).  Shared library: paper_2602_05711_b200/libomnimoe.so.
 *
 * Citations: "PAPER:n" is /root/reference/PAPER.md line n (section/equation
 * named alongside).  Readings of silent or ambiguous passages are numbered Q#
 * and listed in DESIGN.md.
 *
 * Conventions for every entry point
 *  - Every tensor pointer is a DEVICE pointer owned by the caller.  The library
 *    never allocates, frees or synchronises device memory; scratch comes from
 *    the caller's workspace `ws` (size from omnimoe_workspace_size, 256-byte
 *    aligned).  Calls only enqueue work on `stream` and return immediately;
 *    asynchronous faults surface at the caller's next synchronisation.
 *  - Layouts are dense row-major, innermost dimension last; all base pointers
 *    16-byte aligned.
 *  - Element type of x / sub-keys / W / V / MLP weights / y is bf16 when
 *    dims.dtype == OMNIMOE_BF16 and fp32 when OMNIMOE_F32 (correctness mode).
 *  - Validation happens before any launch; on error nothing is enqueued and
 *    omnimoe_last_error() (thread-local) names the offending argument/shape.
 *  - L == 0 (or M == 0) is a successful no-op.
 *  - There is no CPU fallback: a non-sm_100 device returns
 *    OMNIMOE_ERR_UNSUPPORTED.
 */
#ifndef OMNIMOE_H_
#define OMNIMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* omnimoe_stream_t; /* == cudaStream_t */

typedef enum {
  OMNIMOE_OK = 0,
  OMNIMOE_ERR_INVALID_ARGUMENT = 1, /* null required pointer, K<1, h<1, d%8!=0, ... */
  OMNIMOE_ERR_SHAPE = 2,            /* K > N, expert range outside [0,N), M >= 2^31 */
  OMNIMOE_ERR_UNSUPPORTED = 3,      /* not sm_100, unknown dtype / activation / kernel */
  OMNIMOE_ERR_WORKSPACE = 4,        /* ws_bytes below omnimoe_workspace_size() */
  OMNIMOE_ERR_CUDA = 5              /* launch error; text in omnimoe_last_error() */
} omnimoe_status;

enum { OMNIMOE_BF16 = 0, OMNIMOE_F32 = 1 };
/* sigma of the atomic expert (Eq.Atomic).  SILU = z*sigmoid(z)
 * (reading Q1); IDENTITY exists for linearity tests only. */
enum { OMNIMOE_SILU = 0, OMNIMOE_IDENTITY = 1 };
/* Which routed-branch kernel omnimoe_expert_fwd runs: AUTO
 * follows the plan's group size; WARP (expert-major) requires B = 1; GROUP
 * (run-major) requires B > 1.  TOKEN is the paper's ablation "w/o Expert-Centric
 * Scheduling" (Fig. 4a): omnimoe_layer_fwd skips the schedule and each
 * token gathers its own experts' rows (omnimoe_expert_fwd does not accept it). */
enum { OMNIMOE_EXPERT_AUTO = 0, OMNIMOE_EXPERT_WARP = 1, OMNIMOE_EXPERT_GROUP = 2, OMNIMOE_EXPERT_TOKEN = 3,
       OMNIMOE_EXPERT_SLICED = 4, OMNIMOE_EXPERT_DENSE = 5 /* reported by omnimoe_layer_executor only */ };
/* Memory layout of the value table V (the down-projection rows v_n of Eq.WV,
 * PAPER:172-176).  ROWS: [N][d], one row per expert.  SLICED: [d/64][N][64], i.e.
 * the table cut into d/64 column slices of 64 elements, each slice stored
 * expert-major (128 bytes per expert and slice; d % 64 == 0); omnimoe_pack_v converts.  The
 * SLICED executor (AUTO picks it for this layout, bf16 only) evaluates Eq.Grouped
 * in two passes: (Z) the plan's runs compute a = g * sigma(x_l . w_e) for every
 * task with w_e read once per group window; (V) slice by slice, every token
 * gathers the slice of v_e of its tasks and accumulates a * v_e into its output
 * slice.  One band of a slice of V (<= 68 MB) stays L2-resident while all tokens use it,
 * so V is read from HBM once and y_routed is written once, without atomics
 * (DESIGN.md §4.4). */
enum { OMNIMOE_V_ROWS = 0, OMNIMOE_V_SLICED = 1 };
/* workspace query selector */
enum { OMNIMOE_WS_ROUTE = 0, OMNIMOE_WS_SCHEDULE = 1, OMNIMOE_WS_EXPERT = 2, OMNIMOE_WS_LAYER = 3,
       OMNIMOE_WS_ROUTER_BWD = 4, OMNIMOE_WS_MLP_BWD = 5, OMNIMOE_WS_MLP = 6, OMNIMOE_WS_EXPERT_BWD = 7 };

/* How omnimoe_route computes the sub-key logits.  Both give the same bits:
 * logit = RN32(exact dot product x . w) (reading Q9).
 *   EXACT      tcgen05 kind::i8 products of 3 int8 digits per operand (fast);
 *              rows whose exponents span > 22 bits fall back to EXACT_F64.
 *              For K + 1 <= 32 (bf16) the per-half top K+1 is taken inside the
 *              GEMM's epilogue and the logits are not written (N4, PAPER:226-229:
 *              the selection never materialises the score matrix);
 *              the routing result is the same.
 *   EXACT_F64  fp64 double-double dot products on CUDA cores (slow reference). */
enum { OMNIMOE_ROUTER_EXACT = 0, OMNIMOE_ROUTER_EXACT_F64 = 1, OMNIMOE_ROUTER_DENSE = 2 };
/* OMNIMOE_ROUTER_DENSE is the paper's ablation "w/o Cartesian Product Router"
 * (PAPER:395, 414): a standard dense routing projection.  `subkeys` then holds h
 * dense gate tables [h][N][d] (one row per expert, N = n_rows * n_cols); logits =
 * x . W_g^T on the tcgen05 bf16 GEMM with fp32 accumulation (NOT the exact RN32 of
 * Q9), materialised as [L][h][N] fp32 (the "full-dimension logits" the paper blames,
 * PAPER:414); exact top-K of the N logits by (value desc, id asc); gates = softmax
 * over the selected.  bf16 only; ids always in key order. */

/* Layer dimensions.
 *   d          hidden size (multiple of 8)
 *   n_rows     N_r, n_cols N_c: the Cartesian grid, N = N_r * N_c; flat expert id
 *              n = i*N_c + j (row-major, reading Q6)
 *   top_k      K experts per token and head (Eq.TopK), 1 <= K <= N
 *   n_heads    h independent sub-key table pairs over one shared expert pool
 *              (reading Q3); h = 1 is exactly the paper
 *   d_ff       shared-MLP width (0: no shared branch)
 *   router     OMNIMOE_ROUTER_* (ignored in OMNIMOE_F32 mode: always EXACT_F64)
 *   expert_kernel  OMNIMOE_EXPERT_* (a6 kernel choice)
 *   group_size B of Expert-Centric Scheduling: consecutive active
 *              experts per group; 1 = expert-major plan; 0 = library choice
 *              (omnimoe_group_size()).
 *   token_blocks T_b: see below.
 *   v_layout   OMNIMOE_V_ROWS | OMNIMOE_V_SLICED: layout of the V argument of
 *              omnimoe_expert_fwd / omnimoe_layer_fwd (W is always [N][d]).
 *   route_order  order of the K ids omnimoe_route writes per token-head: KEY (by
 *              exact key desc, id asc -- Eq.TopK's ranking) or CANDIDATE (the order
 *              of the Cartesian candidates, row rank then column rank: same set and
 *              gates, no final sort; what omnimoe_layer_fwd uses internally).
 *   v_band_bytes  SLICED pass V: L2 budget of what one pass-V step keeps resident
 *              (one expert band's part of a 64-column slice of V); 0 = library
 *              choice (68 MB).  Determines n_b
 *              (omnimoe_v_bands).  Performance only: results do not depend on it.
 */
enum { OMNIMOE_ORDER_KEY = 0, OMNIMOE_ORDER_CANDIDATE = 1 };
typedef struct {
  int64_t d, n_rows, n_cols, top_k, n_heads, d_ff;
  int32_t dtype;         /* OMNIMOE_BF16 | OMNIMOE_F32 */
  int32_t act;           /* OMNIMOE_SILU | OMNIMOE_IDENTITY */
  int32_t router;        /* OMNIMOE_ROUTER_* */
  int32_t expert_kernel; /* OMNIMOE_EXPERT_* */
  int64_t group_size;    /* B >= 0 */
  int64_t token_blocks;  /* T_b >= 0: the plan is Eq.Sort applied to T_b consecutive token
                          * blocks in turn, so that one block's x and y_routed stay
                          * L2-resident; 1 = the paper's single sort;
                          * 0 = library choice */
  int32_t v_layout;      /* OMNIMOE_V_ROWS | OMNIMOE_V_SLICED */
  int32_t route_order;   /* omnimoe_route output order: OMNIMOE_ORDER_KEY | OMNIMOE_ORDER_CANDIDATE */
  int64_t v_band_bytes;  /* >= 0 */
  int64_t flags;         /* OMNIMOE_FLAG_* (other bits must be 0) */
} omnimoe_dims;
/* flags
 *   OMNIMOE_FLAG_ACT_BF16  omnimoe_expert_fwd (SLICED layout): the routed activations
 *              a_t = g_t sigma(z_t) enter pass V's slice accumulation in bf16 (fp32
 *              accumulation), as omnimoe_layer_fwd always runs it (reading Q21) -- for
 *              callers that round the routed output to bf16 anyway (the expert-parallel
 *              layer's bf16 partials); without it a_t stays fp32. */
enum { OMNIMOE_FLAG_ACT_BF16 = 1 };

/* Expert-centric plan for the local expert range [expert_begin, expert_end)
 * (Eq.Tasks + active compression + Eq.Sort).  n_loc =
 * expert_end - expert_begin; B = the group size resolved from dims.group_size
 * (omnimoe_group_size()).  The tasks of active expert number tau (in ascending
 * id order) belong to group q = floor(tau / B) and are sorted by
 * (q, token) (Eq.Sort); B = 1 is the expert-major order.  Arrays are device
 * memory provided by the caller:
 *   expert_offsets int32[n_loc+1]  task count prefix per local expert; entry
 *                                  n_loc = m_loc, the number of in-range tasks
 *   active         int32[n_loc]    local ids of active experts, ascending
 *   n_active       int32[1]        |E_active| (stays on the device)
 *   sorted_token   int32[M]        token of each task in (q, token) order
 *   sorted_gate    float[M]        its gate g
 *   sorted_expert  int32[M]        its local expert id
 *   run_offsets    int32[M+1]      B > 1 only (nullable for B = 1): first task of
 *                                  each run = the tasks of one token in one group
 *   n_runs         int32[1]        B > 1 only: number of runs P
 * V-order arrays (nullable; required by the SLICED executor; tasks must be
 * sorted by token, which the default token = t / (h*K) is).  The V order sorts
 * the tasks by (token, band) stably, band = local expert id / ceil(n_loc / n_b)
 * with n_b = omnimoe_v_bands(dims, n_loc, n_tok), n_tok = n_tokens if > 0, else
 * ceil(M / (h*K)) in omnimoe_schedule and L in omnimoe_expert_fwd -- the two must
 * agree (they do for the default token = t / (h*K)) (band n_b: outside the range; with
 * n_b = 1 the V order is the task order and out-of-range tasks stay in segment
 * (l, 0) with expert -1):
 *   sorted_task     int32[M]        V-order position of each plan position's task
 *   task_pair       int32[M][2]     per V-order position: (local expert id, -1
 *                                   outside the range; bits of a = g*sigma(z), the
 *                                   scratch of the SLICED executor)
 *   token_offsets   int32[n_tokens*(n_b+1)+1]  start of segment (l, b) at entry
 *                                   l*(n_b+1) + b
 *   n_tokens        number of tokens (input; 0: ceil(M / (h*K)))
 * For B = 1 the segment of local expert e is [expert_offsets[e],
 * expert_offsets[e+1]) with tokens ascending.  Only the first
 * m_loc entries of sorted_* are meaningful (tasks outside the range are not
 * part of the plan). */
typedef struct {
  int32_t* expert_offsets;
  int32_t* sorted_token;
  float* sorted_gate;
  int32_t* active;
  int32_t* n_active;
  int64_t expert_begin, expert_end;
  int32_t* sorted_expert;
  int32_t* run_offsets;
  int32_t* n_runs;
  int32_t* sorted_task;
  int32_t* task_pair;
  int32_t* token_offsets;
  int64_t n_tokens;
} omnimoe_plan;

/* The group size B that omnimoe_schedule / omnimoe_expert_fwd use for dims
 * (dims.group_size if > 0, else the library's choice: 8*N_c experts, at most
 * 64 MB of W/V rows, in bf16 mode; 1 in fp32 mode).  Returns 0 on invalid dims. */
int64_t omnimoe_group_size(const omnimoe_dims* dims);
/* Number of expert bands n_b of the SLICED executor's pass V for a local expert
 * range of n_loc rows and n_tok tokens: pass V sweeps the 64-column slices of V one
 * band at a time; the band's part of a slice (128 bytes per expert) is kept within
 * dims.v_band_bytes (68 MB) so that it stays L2-resident while every token uses it
 * (DESIGN.md §4.4).  Independent of dims.v_layout; 0 on invalid dims. */
int64_t omnimoe_v_bands(const omnimoe_dims* dims, int64_t n_loc, int64_t n_tok);
/* The number of token blocks T_b omnimoe_schedule uses for a batch of L tokens
 * (dims.token_blocks if > 0, else 1; always 1 for B = 1).  Block b holds tokens
 * [b*ceil(L/T_b), (b+1)*ceil(L/T_b)); the plan sorts by (block, q, token). */
int64_t omnimoe_token_blocks(const omnimoe_dims* dims, int64_t L);

/* Bytes of workspace needed by entry point `which` (OMNIMOE_WS_*) for L
 * tokens (ROUTE, EXPERT, LAYER) or M tasks (SCHEDULE: pass M as L). */
omnimoe_status omnimoe_workspace_size(const omnimoe_dims* dims, int64_t L, int which,
                                      size_t* bytes);

/* Cartesian Product Router: Eq.Logits s_r = x W_r, s_c = x W_c
 * with both halves of each head projected from the full x, each logit the fp32
 * rounding of the exact dot product (Q9); exact top-K over the
 * implicit grid S_ij = s_r[i] + s_c[j] (Eq.S; ranking on raw logits is identical
 * to ranking on the log-probabilities, reading Q8), ties between exactly equal
 * keys broken toward the lower flat id (Q7); gates = softmax over the selected
 * keys (Eq.Gate; Q11).
 *   x        [L][d]
 *   subkeys  [h][n_rows + n_cols][d]: row r < n_rows is column r of W_r^h,
 *            row n_rows + c is column c of W_c^h (K-major operand);
 *            [h][N][d] gate rows for OMNIMOE_ROUTER_DENSE
 *   idx      int32 [L][h][K]  flat expert ids, ordered by (key desc, id asc)
 *   gate     float [L][h][K]
 *   score    float [L][h][K]  nullable; p_r[i] + p_c[j] (Eq.LSM + Eq.S)
 * Output is bitwise reproducible and independent of L and batch composition. */
omnimoe_status omnimoe_route(const omnimoe_dims* dims, int64_t L, const void* x,
                             const void* subkeys, int32_t* idx, float* gate, float* score,
                             void* ws, size_t ws_bytes, omnimoe_stream_t stream);

/* Expert-Centric Scheduling: flatten M tasks in token-major order
 * (Eq.Tasks), histogram + exclusive scan over local experts, active-list
 * compaction, group ids q = floor(rank / B), stable LSD radix sort by
 * (token block, q) (Eq.Sort per token block; "radix sort") --
 * stability over the token-major input makes tokens ascend inside each group --
 * and, for B > 1, run detection.  The token of task t must be non-decreasing
 * in t when T_b > 1 (true for the default token = t / (h*K)).
 *   idx   int32[M]  global expert ids of the tasks
 *   gate  float[M]
 *   token int32[M]  nullable: token of task t defaults to t / (h*K)
 *   plan  outputs (see omnimoe_plan); plan->expert_begin/end select the shard
 * Result is bitwise deterministic. */
omnimoe_status omnimoe_schedule(const omnimoe_dims* dims, int64_t M, const int32_t* idx,
                                const float* gate, const int32_t* token, const omnimoe_plan* plan,
                                void* ws, size_t ws_bytes, omnimoe_stream_t stream);

/* Grouped atomic-expert compute + scatter-add (Eq.Grouped, the
 * routed branch of Eq.Assemble): for each task (l, e, g) of the
 * plan: z = x_l . w_e (fp32), a = g * sigma(z), y_routed[l] += a * v_e.
 * B = 1: one warp per active expert reads w_e, v_e once and walks its tokens.
 * B > 1: one warp per run (group q, token l) keeps x_l and the partial y_l in
 * registers over the run's experts and scatter-adds once per run.
 * SLICED (dims.v_layout == OMNIMOE_V_SLICED, B > 1, the plan's task-order arrays
 * set, tasks sorted by token, tokens < L): pass Z over the runs writes
 * plan->task_pair[t][1], pass V writes every y_routed[l] slice once (no atomics,
 * deterministic).
 *   x         [L][d]
 *   W_loc     [n_loc][d]  rows of W for the plan's expert range
 *   V_loc     [n_loc][d] (ROWS) or [d/64][n_loc][64] (SLICED)
 *   y_routed  float [L][d]; overwritten unless accumulate != 0 (then added to)
 * ROWS executors use fp32 atomics: reproducible up to summation order. */
omnimoe_status omnimoe_expert_fwd(const omnimoe_dims* dims, int64_t L, const void* x,
                                  const void* W_loc, const void* V_loc, const omnimoe_plan* plan,
                                  float* y_routed, int accumulate, void* ws, size_t ws_bytes,
                                  omnimoe_stream_t stream);

/* One pass of the SLICED executor, for measurement (pass 1: Z, writes
 * plan->task_pair a-values; pass 2: V, reads them and writes y_routed), run as
 * omnimoe_layer_fwd runs them (pass V takes the a-values in bf16, reading Q21);
 * pass 3 = omnimoe_expert_fwd.  Arguments as omnimoe_expert_fwd. */
omnimoe_status omnimoe_expert_fwd_pass(const omnimoe_dims* dims, int64_t L, const void* x,
                                       const void* W_loc, const void* V_loc, const omnimoe_plan* plan,
                                       float* y_routed, int accumulate, int pass, void* ws,
                                       size_t ws_bytes, omnimoe_stream_t stream);

/* N2: backward of the routed branch for a fixed routing decision
 * (Eq.Assemble, differentiated term by term): with z = x_l . w_e,
 * s = sigma(z), q = dy_l . v_e for each task (l, e, g) of the plan,
 *   dgate[t] = s q                      (task order t = ((l*h)+head)*K + k)
 *   dV_e = sum g s dy_l,  dW_e = sum dz x_l,  dz = g q sigma'(z)
 *   dx_l = sum_t dz_t w_e               (written, or added when accumulate_dx)
 *   x, dy [L][d]; W_loc, V_loc [n_loc][d] (ROWS); W_sliced = omnimoe_pack_v(W_loc)
 *   (the dx pass reads W slice by slice like pass V reads V); plan: the expert-major
 *   plan (group size 1) with its V-order arrays and ONE band (dims.v_band_bytes >=
 *   128 n_loc; otherwise OMNIMOE_ERR_UNSUPPORTED); dW_act, dV_act fp32
 *   [n_loc][d]: row tau = the expert plan->active[tau] (tau < n_active; other rows
 *   untouched); dgate fp32 [M].  bf16, d % 64 == 0, d <= 2048; no atomics (every
 *   expert row and every dx slice is owned by one warp; summation orders are fixed).
 *   ws: omnimoe_workspace_size(dims, L, OMNIMOE_WS_EXPERT_BWD) bytes. */
omnimoe_status omnimoe_expert_bwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* W_loc,
                                  const void* V_loc, const void* W_sliced, const omnimoe_plan* plan,
                                  const void* dy, float* dx, float* dW_act, float* dV_act, float* dgate,
                                  int accumulate_dx, void* ws, size_t ws_bytes, omnimoe_stream_t stream);

/* N2, router part: gradients through the gates (softmax over the K selected keys,
 * Eq.Gate) and the sub-key logits (key = s_r[i] + s_c[j], s = x . sub,
 * Eq.S / Eq.Logits) with the selection held fixed:
 *   dkappa_k = g_k (dgate_k - sum_j g_j dgate_j);  ds_r[i] += dkappa, ds_c[j] += dkappa
 *   dsub[h][r] = sum_l ds[l][h][r] x_l   (fp32 [h][N_r+N_c][d], overwritten)
 *   dx_l (+)= sum_{h,r} ds[l][h][r] sub[h][r]   (fp32 [L][d]; added when accumulate_dx)
 *   idx, gate [L][h][K]: the forward's routing (any order); dgate [L][h][K] (from
 *   omnimoe_expert_bwd).  ds is rounded to bf16 for the tcgen05 GEMMs.
 *   ws: omnimoe_workspace_size(OMNIMOE_WS_ROUTER_BWD). */
omnimoe_status omnimoe_router_bwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* subkeys,
                                  const int32_t* idx, const float* gate, const float* dgate, float* dx,
                                  int accumulate_dx, float* dsubkeys, void* ws, size_t ws_bytes,
                                  omnimoe_stream_t stream);

/* N2, shared MLP (reading Q2): with G|U = x W_gu^T, H = SiLU(G) U:
 *   dw_down = dy^T H (fp32 [d][d_ff]), dw_gate_up = [dG|dU]^T x (fp32 [2 d_ff][d]),
 *   dx (+)= [dG|dU] W_gu, where dU = dH SiLU(G), dG = dH U SiLU'(G), dH = dy W_down.
 *   bf16 operands on the tcgen05 GEMM engine, fp32 results.
 *   ws: omnimoe_workspace_size(OMNIMOE_WS_MLP_BWD). */
omnimoe_status omnimoe_shared_mlp_bwd(const omnimoe_dims* dims, int64_t L, const void* x, const void* w_gate_up,
                                      const void* w_down, const void* dy, float* dx, int accumulate_dx,
                                      float* dw_gate_up, float* dw_down, void* ws, size_t ws_bytes,
                                      omnimoe_stream_t stream);

/* V [n][d] (OMNIMOE_V_ROWS) -> V_sliced [d/64][n][64] (OMNIMOE_V_SLICED): a
 * one-time weight re-layout (no arithmetic; bit-exact copy), d % 64 == 0.
 * n = number of expert rows in the table (N, or n_loc for a shard). */
omnimoe_status omnimoe_pack_v(const omnimoe_dims* dims, int64_t n, const void* V, void* V_sliced,
                              omnimoe_stream_t stream);

/* Shared dense MLP (SwiGLU without biases, reading Q2) plus
 * combine (Eq.MoE):
 *   H = silu(x W_gate^T) * (x W_up^T)  (in OMNIMOE_BF16 mode a bf16 pair hi + lo, ~16
 *                                       significant bits, when d_ff % 64 == 0, else bf16)
 *   y = H W_down^T + y_routed           (y_routed nullable -> treated as 0)
 *   w_gate_up [2*d_ff][d] (gate rows, then up rows), w_down [d][d_ff],
 *   y [L][d] (bf16 or fp32 per dtype). */
omnimoe_status omnimoe_shared_mlp(const omnimoe_dims* dims, int64_t L, const void* x,
                                  const void* w_gate_up, const void* w_down, const float* y_routed,
                                  void* y, void* ws, size_t ws_bytes, omnimoe_stream_t stream);
/*   ws: omnimoe_workspace_size(dims, L, OMNIMOE_WS_MLP) bytes (holds H). */
/* The same two GEMMs as separate calls, so that GEMM-1 (which needs only x) can run
 * while the routed branch is still in flight (the expert-parallel driver overlaps it
 * with the dispatch all-to-all):
 *   omnimoe_shared_mlp_hidden: H = silu(x W_gate^T) * (x W_up^T) into H (H_bytes >=
 *     omnimoe_workspace_size(dims, L, OMNIMOE_WS_MLP); layout opaque);
 *   omnimoe_shared_mlp_out:    y = H W_down^T + y_routed (y_routed nullable). */
omnimoe_status omnimoe_shared_mlp_hidden(const omnimoe_dims* dims, int64_t L, const void* x, const void* w_gate_up,
                                         void* H, size_t H_bytes, omnimoe_stream_t stream);
omnimoe_status omnimoe_shared_mlp_out(const omnimoe_dims* dims, int64_t L, const void* H, size_t H_bytes,
                                      const void* w_down, const float* y_routed, void* y, omnimoe_stream_t stream);

/* The paper's ablation "w/o Expert-Centric Scheduling": the routed
 * branch token by token straight from the routing decision (idx, gate [L][h*K],
 * global ids), every task gathering its own w_e and v_e rows; y_routed[l] written
 * once (added to when accumulate != 0).  V in the ROWS layout; bf16, d % 256 == 0. */
omnimoe_status omnimoe_expert_fwd_tokens(const omnimoe_dims* dims, int64_t L, const void* x, const void* W,
                                         const void* V, const int32_t* idx, const float* gate,
                                         float* y_routed, int accumulate, omnimoe_stream_t stream);

/* The routed branch as two dense tcgen05 GEMMs (the executor omnimoe_layer_fwd picks
 * when one head selects K >= N/40 experts and eta >= 32): Z = x W^T [L][N] fp32; A = gate * sigma(Z) on the selected cells, 0
 * elsewhere (bf16); y_routed = A V (written, fp32).  idx, gate [L][h*K] global ids;
 * one head; V in the ROWS layout; ws: omnimoe_dense_workspace_size(). */
size_t omnimoe_dense_workspace_size(const omnimoe_dims* dims, int64_t L);
omnimoe_status omnimoe_expert_fwd_dense(const omnimoe_dims* dims, int64_t L, const void* x, const void* W,
                                        const void* V, const int32_t* idx, const float* gate, float* y_routed,
                                        void* ws, size_t ws_bytes, omnimoe_stream_t stream);

/* The routed-branch executor omnimoe_layer_fwd runs for dims and L tokens
 * (OMNIMOE_EXPERT_*; -1 on invalid dims).  With expert_kernel AUTO: SLICED for the
 * SLICED layout; for the ROWS layout TOKEN when eta = M / E|E_active| < 2 under
 * uniform routing (then no expert is shared by two tasks and Expert-Centric
 * Scheduling has nothing to reuse -- measured faster); DENSE when
 * one head selects K >= N/40 experts and eta >= 32 (the routed branch as two tcgen05
 * GEMMs, Z = x W^T, A = gate * sigma(Z) on the selected cells, y = A V); else GROUP. */
int32_t omnimoe_layer_executor(const omnimoe_dims* dims, int64_t L);

/* Whole layer forward (Eq.MoE / Eq.Assemble):
 * route -> schedule (full expert range) -> expert_fwd -> shared MLP + combine.
 *   W          [N][d]
 *   V          [N][d] or, for dims.v_layout == OMNIMOE_V_SLICED, [d/64][N][64]
 *   w_gate_up, w_down  as in omnimoe_shared_mlp (ignored when d_ff == 0)
 *   y          [L][d]
 *   idx_out, gate_out  nullable copies of the routing decision [L][h][K]; the same
 *              set and gates as omnimoe_route, but (for K + 1 > 32) in the order of the
 *              Cartesian candidates (row rank, then column rank) instead of by key --
 *              the layer never needs the sort
 * Precision: the routed activations a_t = g_t sigma(z_t) enter the SLICED executor's
 * slice accumulation in bf16 (fp32 accumulation; reading Q21 -- the output is bf16);
 * omnimoe_expert_fwd keeps them in fp32. */
omnimoe_status omnimoe_layer_fwd(const omnimoe_dims* dims, int64_t L, const void* x,
                                 const void* subkeys, const void* W, const void* V,
                                 const void* w_gate_up, const void* w_down, void* y,
                                 int32_t* idx_out, float* gate_out, void* ws, size_t ws_bytes,
                                 omnimoe_stream_t stream);

/* omnimoe_layer_fwd for activations in (pinned) HOST memory, with the transfers
 * overlapped: x is copied to the caller's device buffer x_dev in `chunks` token
 * chunks on copy_stream while the chunks already copied are routed on stream (the
 * router is per token and batch-independent: the routing is bit-identical); the
 * schedule and routed branch run on the whole batch; the shared MLP's second GEMM
 * (+ combine) runs chunk by chunk and each chunk of y (device buffer y_dev) is copied
 * to y_host on copy_stream while the next is computed.  The call is complete on
 * `stream` once y_host holds the result.  Chunks are whole multiples of 128 tokens.
 *   x_host, y_host [L][d] host (pinned for overlap); x_dev, y_dev [L][d] device;
 *   copy_stream: a second stream of the caller's; ws as omnimoe_layer_fwd. */
omnimoe_status omnimoe_layer_fwd_host(const omnimoe_dims* dims, int64_t L, const void* x_host, void* x_dev,
                                      const void* subkeys, const void* W, const void* V,
                                      const void* w_gate_up, const void* w_down, void* y_dev, void* y_host,
                                      int chunks, void* ws, size_t ws_bytes, omnimoe_stream_t stream,
                                      omnimoe_stream_t copy_stream);

/* The sub-key logits of the route call, for measurement and parity:
 * logits float [L][h][n_rows+n_cols].  method 0: the route path (dims.router);
 * 1: exact fp64 double-double kernel; 2: bf16 tcgen05 GEMM with fp32
 * accumulation (NOT exact -- only to measure what exactness costs).
 * ws: at least omnimoe_workspace_size(OMNIMOE_WS_ROUTE) bytes. */
omnimoe_status omnimoe_router_logits(const omnimoe_dims* dims, int64_t L, const void* x,
                                     const void* subkeys, float* logits, int method, void* ws,
                                     size_t ws_bytes, omnimoe_stream_t stream);

/* Plain GEMM on the library's tcgen05 engine (bf16 in, fp32 out):
 * C[M][N] = A[M][K] . B[N][K]^T.  Exposed for engine tests / roofline. */
omnimoe_status omnimoe_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, const void* B,
                                 float* C, omnimoe_stream_t stream);

/* ---- Expert parallelism over R ranks ----------
 * Rank r owns flat expert ids [r*n_per, (r+1)*n_per), n_per = N / R (whole grid
 * rows since n = i*N_c + j), and L of the batch's tokens.  The collectives
 * themselves (NCCL all-to-all over NVLink) are issued by the caller
 * (paper_2602_05711_b200/distributed.py); these calls pack, unpack and combine.
 *
 * omnimoe_ep_pack: from the routing decision idx/gate [L][h*K] of the local
 * tokens, write for every destination s (in rank order):
 *   x_send   [sum_s T_s][d]  each local token with >= 1 task on s, once, tokens
 *                            ascending ("slot" = row within s's block)
 *   rec_send int32 [sum_s M_s][3]  per task on s: (id - s*n_per, gate bits, slot)
 *   inv      int32 [R][L]    slot of token l in s's block, -1 if none
 *   offsets  int32 [2R+2]    token block starts [0..R] (R+1 entries), then task
 *                            block starts [0..R]
 *   counts   int64 [R][2]    (nullable) rows and records per destination -- the
 *                            split sizes of the all-to-alls, ready to be exchanged
 *                            device to device (one host read per forward for both
 *                            directions)
 * Sizes are bounded by R*L rows and L*h*K records.  ws: omnimoe_ep_pack_workspace_size. */
omnimoe_status omnimoe_ep_pack_workspace_size(int64_t L, int32_t R, size_t* bytes);
omnimoe_status omnimoe_ep_pack(const omnimoe_dims* dims, int64_t L, int32_t R, const void* x,
                               const int32_t* idx, const float* gate, void* x_send, int32_t* rec_send,
                               int32_t* inv, int32_t* offsets, int64_t* counts, void* ws, size_t ws_bytes,
                               omnimoe_stream_t stream);
/* Received records (concatenated by source rank; task_off/tok_off int64 [R+1] are
 * the per-source block starts of the received records / x rows, device memory)
 * -> task arrays for omnimoe_schedule over the local expert range [0, n_per):
 * ids (local expert id), gate, token (= row of the received x buffer). */
omnimoe_status omnimoe_ep_unpack(int64_t M, int32_t R, const int32_t* rec, const int64_t* task_off,
                                 const int64_t* tok_off, int32_t* ids, float* gate, int32_t* token,
                                 omnimoe_stream_t stream);
/* The partial output rows of a shard, fp32 [rows][d] -> bf16 [rows][d] (round to
 * nearest even) for the return all-to-all: half the bytes of fp32. */
omnimoe_status omnimoe_ep_partials(int64_t rows, const omnimoe_dims* dims, const float* y_part, void* y_bf16,
                                   omnimoe_stream_t stream);
/* y_routed[l] = sum over s = 0..R-1 (in that order) of y_ret[tok_off[s] + inv[s][l]]
 * (skipped where inv = -1), accumulated in fp32: the returned partial rows [rows][d],
 * bf16 (y_ret_bf16 != 0, from omnimoe_ep_partials) or fp32. */
omnimoe_status omnimoe_ep_combine(const omnimoe_dims* dims, int64_t L, int32_t R, const void* y_ret,
                                  int32_t y_ret_bf16, const int32_t* inv, const int64_t* tok_off, float* y_routed,
                                  omnimoe_stream_t stream);

/* Load metrics of a plan's routing (after PKM / PEER): with c_e the
 * task count of local expert e (plan->expert_offsets), M = sum c_e, n = n_loc and
 * z_e = c_e / M:  stats[0] = Expert Usage = |{e : c_e > 0}| / n,
 *                 stats[1] = Unevenness = D_KL(z || U) = sum_{c_e > 0} z_e log(n z_e).
 * stats: device fp64[2]; ws: omnimoe_load_stats_workspace_size() bytes.  Summation
 * order is fixed (deterministic). */
omnimoe_status omnimoe_load_stats(const omnimoe_plan* plan, double* stats, void* ws, size_t ws_bytes,
                                  omnimoe_stream_t stream);
size_t omnimoe_load_stats_workspace_size(void);

/* Number of kernel launches the last successful call on this thread enqueued. */
int omnimoe_last_launch_count(void);

const char* omnimoe_status_string(omnimoe_status s);
const char* omnimoe_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* OMNIMOE_H_ */
