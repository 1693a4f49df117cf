"""Thin ctypes binding over libomnimoe.so (include/omnimoe.h).

Argument marshalling only: every step of the layer runs in the library's CUDA
kernels.  Tensors must be CUDA, contiguous, of the dtype the dims declare; the
calls enqueue on torch's current stream.  There is no CPU fallback: if the
shared library is missing or the device is not sm_100a, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# OMNIMOE_LIB: another build of the same library (the measurement build of tools/ sweeps)
LIB_PATH = os.environ.get("OMNIMOE_LIB") or os.path.join(_PKG, "libomnimoe.so")

BF16, F32 = 0, 1
SILU, IDENTITY = 0, 1
EXPERT_AUTO, EXPERT_WARP, EXPERT_GROUP, EXPERT_TOKEN, EXPERT_SLICED, EXPERT_DENSE = 0, 1, 2, 3, 4, 5
V_ROWS, V_SLICED = 0, 1
ORDER_KEY, ORDER_CANDIDATE = 0, 1
FLAG_ACT_BF16 = 1
ROUTER_EXACT, ROUTER_EXACT_F64, ROUTER_DENSE = 0, 1, 2
LOGITS_ROUTE, LOGITS_EXACT_F64, LOGITS_BF16_FAST = 0, 1, 2
WS_ROUTE, WS_SCHEDULE, WS_EXPERT, WS_LAYER, WS_ROUTER_BWD, WS_MLP_BWD, WS_MLP, WS_EXPERT_BWD = 0, 1, 2, 3, 4, 5, 6, 7


class OmniMoEError(RuntimeError):
    pass


class Dims(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int64), ("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64),
                ("top_k", ctypes.c_int64), ("n_heads", ctypes.c_int64), ("d_ff", ctypes.c_int64),
                ("dtype", ctypes.c_int32), ("act", ctypes.c_int32), ("router", ctypes.c_int32),
                ("expert_kernel", ctypes.c_int32), ("group_size", ctypes.c_int64),
                ("token_blocks", ctypes.c_int64), ("v_layout", ctypes.c_int32), ("route_order", ctypes.c_int32),
                ("v_band_bytes", ctypes.c_int64), ("flags", ctypes.c_int64)]


class Plan(ctypes.Structure):
    _fields_ = [("expert_offsets", ctypes.c_void_p), ("sorted_token", ctypes.c_void_p),
                ("sorted_gate", ctypes.c_void_p), ("active", ctypes.c_void_p),
                ("n_active", ctypes.c_void_p), ("expert_begin", ctypes.c_int64),
                ("expert_end", ctypes.c_int64), ("sorted_expert", ctypes.c_void_p),
                ("run_offsets", ctypes.c_void_p), ("n_runs", ctypes.c_void_p),
                ("sorted_task", ctypes.c_void_p), ("task_pair", ctypes.c_void_p), ("token_offsets", ctypes.c_void_p),
                ("n_tokens", ctypes.c_int64)]


EXPORTS = ["omnimoe_workspace_size", "omnimoe_route", "omnimoe_schedule", "omnimoe_expert_fwd",
           "omnimoe_shared_mlp", "omnimoe_layer_fwd", "omnimoe_router_logits", "omnimoe_gemm_bf16",
           "omnimoe_last_launch_count", "omnimoe_status_string", "omnimoe_last_error",
           "omnimoe_group_size", "omnimoe_token_blocks", "omnimoe_ep_pack_workspace_size",
           "omnimoe_ep_pack", "omnimoe_ep_unpack", "omnimoe_ep_combine", "omnimoe_pack_v",
           "omnimoe_v_bands", "omnimoe_expert_fwd_pass", "omnimoe_load_stats",
           "omnimoe_load_stats_workspace_size", "omnimoe_expert_fwd_tokens", "omnimoe_layer_executor",
           "omnimoe_expert_bwd", "omnimoe_router_bwd", "omnimoe_shared_mlp_bwd", "omnimoe_layer_fwd_host",
           "omnimoe_expert_fwd_dense", "omnimoe_dense_workspace_size", "omnimoe_ep_partials",
           "omnimoe_shared_mlp_hidden", "omnimoe_shared_mlp_out"]

_lib = None


def load(path: str = LIB_PATH):
    """Load libomnimoe.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OmniMoEError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    V, I64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    PD, PP = ctypes.POINTER(Dims), ctypes.POINTER(Plan)
    sig = {
        "omnimoe_workspace_size": [PD, I64, I32, ctypes.POINTER(ctypes.c_size_t)],
        "omnimoe_route": [PD, I64, V, V, V, V, V, V, SZ, V],
        "omnimoe_schedule": [PD, I64, V, V, V, PP, V, SZ, V],
        "omnimoe_expert_fwd": [PD, I64, V, V, V, PP, V, I32, V, SZ, V],
        "omnimoe_expert_fwd_pass": [PD, I64, V, V, V, PP, V, I32, I32, V, SZ, V],
        "omnimoe_shared_mlp": [PD, I64, V, V, V, V, V, V, SZ, V],
        "omnimoe_layer_fwd": [PD, I64, V, V, V, V, V, V, V, V, V, V, SZ, V],
        "omnimoe_router_logits": [PD, I64, V, V, V, I32, V, SZ, V],
        "omnimoe_gemm_bf16": [I64, I64, I64, V, V, V, V],
        "omnimoe_ep_pack_workspace_size": [I64, I32, ctypes.POINTER(ctypes.c_size_t)],
        "omnimoe_ep_pack": [PD, I64, I32, V, V, V, V, V, V, V, V, V, SZ, V],
        "omnimoe_ep_unpack": [I64, I32, V, V, V, V, V, V, V],
        "omnimoe_ep_partials": [I64, PD, V, V, V],
        "omnimoe_ep_combine": [PD, I64, I32, V, I32, V, V, V, V],
        "omnimoe_shared_mlp_hidden": [PD, I64, V, V, V, SZ, V],
        "omnimoe_shared_mlp_out": [PD, I64, V, SZ, V, V, V, V],
        "omnimoe_pack_v": [PD, I64, V, V, V],
        "omnimoe_load_stats": [PP, V, V, SZ, V],
        "omnimoe_expert_fwd_tokens": [PD, I64, V, V, V, V, V, V, I32, V],
        "omnimoe_expert_bwd": [PD, I64, V, V, V, V, PP, V, V, V, V, V, I32, V, SZ, V],
        "omnimoe_router_bwd": [PD, I64, V, V, V, V, V, V, I32, V, V, SZ, V],
        "omnimoe_expert_fwd_dense": [PD, I64, V, V, V, V, V, V, V, SZ, V],
        "omnimoe_layer_fwd_host": [PD, I64, V, V, V, V, V, V, V, V, V, I32, V, SZ, V, V],
        "omnimoe_shared_mlp_bwd": [PD, I64, V, V, V, V, V, I32, V, V, V, SZ, V],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.omnimoe_last_launch_count.restype = ctypes.c_int
    lib.omnimoe_group_size.argtypes = [PD]
    lib.omnimoe_group_size.restype = ctypes.c_int64
    lib.omnimoe_dense_workspace_size.argtypes = [PD, ctypes.c_int64]
    lib.omnimoe_dense_workspace_size.restype = ctypes.c_size_t
    lib.omnimoe_layer_executor.argtypes = [PD, ctypes.c_int64]
    lib.omnimoe_layer_executor.restype = ctypes.c_int32
    lib.omnimoe_load_stats_workspace_size.restype = ctypes.c_size_t
    lib.omnimoe_load_stats_workspace_size.argtypes = []
    lib.omnimoe_v_bands.argtypes = [PD, ctypes.c_int64, ctypes.c_int64]
    lib.omnimoe_v_bands.restype = ctypes.c_int64
    lib.omnimoe_token_blocks.argtypes = [PD, ctypes.c_int64]
    lib.omnimoe_token_blocks.restype = ctypes.c_int64
    lib.omnimoe_status_string.restype = ctypes.c_char_p
    lib.omnimoe_status_string.argtypes = [ctypes.c_int]
    lib.omnimoe_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


LAUNCHES = 0  # kernels enqueued by this process through the library (omnimoe_last_launch_count)


def _check(status: int, what: str):
    global LAUNCHES
    lib = load()
    if status != 0:
        raise OmniMoEError(f"{what}: {lib.omnimoe_status_string(status).decode()}: "
                           f"{lib.omnimoe_last_error().decode()}")
    LAUNCHES += lib.omnimoe_last_launch_count()


def last_launch_count() -> int:
    return load().omnimoe_last_launch_count()


@dataclass
class LayerDims:
    d: int
    n_rows: int
    n_cols: int
    top_k: int
    n_heads: int = 1
    d_ff: int = 0
    dtype: int = BF16
    act: int = SILU
    router: int = ROUTER_EXACT
    expert_kernel: int = EXPERT_AUTO
    group_size: int = 0
    token_blocks: int = 0
    v_layout: int = V_ROWS
    route_order: int = ORDER_KEY
    v_band_bytes: int = 0
    flags: int = 0  # FLAG_ACT_BF16: omnimoe_expert_fwd takes the activations in bf16 (reading Q21)

    @property
    def N(self) -> int:
        return self.n_rows * self.n_cols

    @property
    def router_rows(self) -> int:
        """Rows of each head's router table: N_r + N_c sub-keys, or N gate rows for the
        dense-router ablation."""
        return self.N if self.router == ROUTER_DENSE else self.n_rows + self.n_cols

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == BF16 else torch.float32

    def c(self) -> Dims:
        return Dims(self.d, self.n_rows, self.n_cols, self.top_k, self.n_heads, self.d_ff,
                    self.dtype, self.act, self.router, self.expert_kernel, self.group_size,
                    self.token_blocks, self.v_layout, self.route_order, self.v_band_bytes, self.flags)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _req(t, name, dtype=None, numel=None):
    if t is None:
        raise OmniMoEError(f"{name} is required")
    if not t.is_cuda:
        raise OmniMoEError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise OmniMoEError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise OmniMoEError(f"{name} must be {dtype}, got {t.dtype}")
    if numel is not None and t.numel() != numel:
        raise OmniMoEError(f"{name} must have {numel} elements, got {t.numel()}")
    return t


def workspace_size(dims: LayerDims, L: int, which: int) -> int:
    out = ctypes.c_size_t(0)
    dc = dims.c()
    _check(load().omnimoe_workspace_size(ctypes.byref(dc), L, which, ctypes.byref(out)), "workspace_size")
    return out.value


def workspace(dims: LayerDims, L: int, which: int, device=None) -> torch.Tensor:
    return torch.empty(max(workspace_size(dims, L, which), 1), dtype=torch.uint8,
                       device=device or torch.cuda.current_device())


def route(dims: LayerDims, x, subkeys, ws=None, want_score=True):
    L = x.shape[0]
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(subkeys, "subkeys", dims.torch_dtype, dims.n_heads * dims.router_rows * dims.d)
    K, h = dims.top_k, dims.n_heads
    idx = torch.empty((L, h, K), dtype=torch.int32, device=x.device)
    gate = torch.empty((L, h, K), dtype=torch.float32, device=x.device)
    score = torch.empty((L, h, K), dtype=torch.float32, device=x.device) if want_score else None
    ws = ws if ws is not None else workspace(dims, L, WS_ROUTE, x.device)
    dc = dims.c()
    _check(load().omnimoe_route(ctypes.byref(dc), L, _ptr(x), _ptr(subkeys), _ptr(idx), _ptr(gate),
                                _ptr(score), _ptr(ws), ws.numel(), _stream()), "route")
    return idx, gate, score


def group_size(dims: LayerDims) -> int:
    """The group size B the library uses for these dims."""
    dc = dims.c()
    return int(load().omnimoe_group_size(ctypes.byref(dc)))


def token_blocks(dims: LayerDims, L: int) -> int:
    """The number of token blocks T_b the schedule uses for L tokens."""
    dc = dims.c()
    return int(load().omnimoe_token_blocks(ctypes.byref(dc), L))


def v_bands(dims: LayerDims, n_loc: int, n_tok: int) -> int:
    """Expert bands of the SLICED executor's pass V for n_loc local experts and n_tok tokens."""
    dc = dims.c()
    return int(load().omnimoe_v_bands(ctypes.byref(dc), n_loc, n_tok))


def new_plan(n_loc: int, M: int, device, expert_begin: int = 0, n_tokens: int = 0, dims: LayerDims = None):
    """Plan buffers (omnimoe_plan).  n_tokens: tokens of the task list (0: M / (h*K));
    the V-order arrays of the SLICED executor are always allocated (for dims' bands)."""
    n_tok = n_tokens if n_tokens > 0 else (-(-M // (dims.n_heads * dims.top_k)) if dims is not None else M)
    nb = v_bands(dims, n_loc, max(n_tok, 1)) if dims is not None else 1
    t = dict(sorted_task=torch.empty(max(M, 1), dtype=torch.int32, device=device),
             task_pair=torch.empty((max(M, 1), 2), dtype=torch.int32, device=device),
             token_offsets=torch.empty(max(n_tokens, M, 1) * (nb + 1) + 1, dtype=torch.int32, device=device),
             n_tokens=n_tokens,
expert_offsets=torch.empty(n_loc + 1, dtype=torch.int32, device=device),
             sorted_token=torch.empty(max(M, 1), dtype=torch.int32, device=device),
             sorted_gate=torch.empty(max(M, 1), dtype=torch.float32, device=device),
             sorted_expert=torch.empty(max(M, 1), dtype=torch.int32, device=device),
             run_offsets=torch.empty(M + 1, dtype=torch.int32, device=device),
             n_runs=torch.zeros(1, dtype=torch.int32, device=device),
             active=torch.empty(max(n_loc, 1), dtype=torch.int32, device=device),
             n_active=torch.empty(1, dtype=torch.int32, device=device),
             expert_begin=expert_begin, expert_end=expert_begin + n_loc)
    return t


def _cplan(p) -> Plan:
    return Plan(p["expert_offsets"].data_ptr(), p["sorted_token"].data_ptr(), p["sorted_gate"].data_ptr(),
                p["active"].data_ptr(), p["n_active"].data_ptr(), p["expert_begin"], p["expert_end"],
                p["sorted_expert"].data_ptr(), p["run_offsets"].data_ptr(), p["n_runs"].data_ptr(),
                p["sorted_task"].data_ptr(), p["task_pair"].data_ptr(),
                p["token_offsets"].data_ptr(), p["n_tokens"])


def schedule(dims: LayerDims, idx, gate, token=None, expert_begin=0, expert_end=None, plan=None, ws=None,
             n_tokens=0):
    """Expert-centric plan (a4 + a5) of the tasks (idx, gate) over the expert range.
    n_tokens: number of tokens when `token` is given (tasks sorted by token)."""
    M = idx.numel()
    _req(idx, "idx", torch.int32)
    _req(gate, "gate", torch.float32, M)
    if token is not None:
        _req(token, "token", torch.int32, M)
    expert_end = dims.N if expert_end is None else expert_end
    n_loc = expert_end - expert_begin
    plan = plan or new_plan(n_loc, M, idx.device, expert_begin, n_tokens, dims)
    ws = ws if ws is not None else torch.empty(max(workspace_size(dims, M, WS_SCHEDULE), 1),
                                               dtype=torch.uint8, device=idx.device)
    dc, cp = dims.c(), _cplan(plan)
    _check(load().omnimoe_schedule(ctypes.byref(dc), M, _ptr(idx), _ptr(gate), _ptr(token),
                                   ctypes.byref(cp), _ptr(ws), ws.numel(), _stream()), "schedule")
    return plan


def load_stats(plan):
    """(Expert Usage, Unevenness) of a plan's routing as a device
    fp64 tensor [2] (omnimoe_load_stats)."""
    lib = load()
    dev = plan["expert_offsets"].device
    out = torch.empty(2, dtype=torch.float64, device=dev)
    ws = torch.empty(lib.omnimoe_load_stats_workspace_size(), dtype=torch.uint8, device=dev)
    cp = _cplan(plan)
    _check(lib.omnimoe_load_stats(ctypes.byref(cp), _ptr(out), _ptr(ws), ws.numel(), _stream()), "load_stats")
    return out


def expert_bwd(dims: LayerDims, x, W_loc, V_loc, W_sliced, plan, dy, dx=None, accumulate_dx=False, ws=None):
    """N2: routed-branch backward for the plan's routing (omnimoe_expert_bwd).
    Returns (dx [L][d], dW_act, dV_act [n_active][d] in plan['active'] order, dgate [M])."""
    L = x.shape[0]
    n_loc = plan["expert_end"] - plan["expert_begin"]
    M = plan["sorted_task"].numel()
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(dy, "dy", dims.torch_dtype, L * dims.d)
    _req(W_loc, "W_loc", dims.torch_dtype, n_loc * dims.d)
    _req(V_loc, "V_loc", dims.torch_dtype, n_loc * dims.d)
    _req(W_sliced, "W_sliced", dims.torch_dtype, n_loc * dims.d)
    dev = x.device
    if dx is None:
        dx = torch.empty((L, dims.d), dtype=torch.float32, device=dev)
        accumulate_dx = False
    dW = torch.empty((n_loc, dims.d), dtype=torch.float32, device=dev)
    dV = torch.empty((n_loc, dims.d), dtype=torch.float32, device=dev)
    dg = torch.empty(max(M, 1), dtype=torch.float32, device=dev)
    ws = ws if ws is not None else workspace(dims, L, WS_EXPERT_BWD, dev)
    dc, cp = dims.c(), _cplan(plan)
    _check(load().omnimoe_expert_bwd(ctypes.byref(dc), L, _ptr(x), _ptr(W_loc), _ptr(V_loc), _ptr(W_sliced),
                                     ctypes.byref(cp), _ptr(dy), _ptr(dx), _ptr(dW), _ptr(dV), _ptr(dg),
                                     int(accumulate_dx), _ptr(ws), ws.numel(), _stream()), "expert_bwd")
    na = int(plan["n_active"].item())
    return dx, dW[:na], dV[:na], dg[:M]


def router_bwd(dims: LayerDims, x, subkeys, idx, gate, dgate, dx=None, accumulate_dx=False):
    """N2 router part (omnimoe_router_bwd) -> (dx [L][d] fp32, dsubkeys [h][R][d] fp32)."""
    L = x.shape[0]
    dev = x.device
    if dx is None:
        dx = torch.empty((L, dims.d), dtype=torch.float32, device=dev)
        accumulate_dx = False
    dsub = torch.empty((dims.n_heads, dims.n_rows + dims.n_cols, dims.d), dtype=torch.float32, device=dev)
    ws = workspace(dims, L, WS_ROUTER_BWD, dev)
    dc = dims.c()
    _check(load().omnimoe_router_bwd(ctypes.byref(dc), L, _ptr(x), _ptr(subkeys), _ptr(idx.contiguous()),
                                     _ptr(gate.contiguous()), _ptr(dgate.contiguous()), _ptr(dx),
                                     int(accumulate_dx), _ptr(dsub), _ptr(ws), ws.numel(), _stream()), "router_bwd")
    return dx, dsub


def shared_mlp_bwd(dims: LayerDims, x, w_gate_up, w_down, dy, dx=None, accumulate_dx=False):
    """N2 shared-MLP part (omnimoe_shared_mlp_bwd) -> (dx, dw_gate_up, dw_down), fp32."""
    L = x.shape[0]
    dev = x.device
    if dx is None:
        dx = torch.empty((L, dims.d), dtype=torch.float32, device=dev)
        accumulate_dx = False
    dgu = torch.empty((2 * dims.d_ff, dims.d), dtype=torch.float32, device=dev)
    ddn = torch.empty((dims.d, dims.d_ff), dtype=torch.float32, device=dev)
    ws = workspace(dims, L, WS_MLP_BWD, dev)
    dc = dims.c()
    _check(load().omnimoe_shared_mlp_bwd(ctypes.byref(dc), L, _ptr(x), _ptr(w_gate_up), _ptr(w_down), _ptr(dy),
                                         _ptr(dx), int(accumulate_dx), _ptr(dgu), _ptr(ddn), _ptr(ws), ws.numel(),
                                         _stream()), "shared_mlp_bwd")
    return dx, dgu, ddn


def bwd_dims(dims: LayerDims) -> LayerDims:
    """The dims the backward's plan is scheduled with (and omnimoe_expert_bwd called with):
    group size 1 and one V band, so that the plan's V order is the task order."""
    return _replace(dims, group_size=1, v_band_bytes=max(dims.v_band_bytes, 128 * dims.N + 1))


def layer_bwd(dims: LayerDims, x, subkeys, W, V, W_sliced, w_gate_up, w_down, idx, gate, plan, dy):
    """N2: the layer's backward for the forward's routing decision (idx, gate [L][h][K],
    the plan of those tasks scheduled with bwd_dims(dims)): routed branch (omnimoe_expert_bwd), router
    gates (omnimoe_router_bwd) and shared MLP (omnimoe_shared_mlp_bwd), dx summed over the
    three.  Returns dict(dx, dsubkeys, dW_act, dV_act, active, dgate, dw_gate_up, dw_down)."""
    rd = bwd_dims(dims)
    dx, dW, dV, dg = expert_bwd(rd, x, W, V, W_sliced, plan, dy)
    _, dsub = router_bwd(dims, x, subkeys, idx, gate, dg.reshape(gate.shape), dx=dx, accumulate_dx=True)
    out = dict(dx=dx, dsubkeys=dsub, dW_act=dW, dV_act=dV, active=plan["active"][:dW.shape[0]], dgate=dg)
    if dims.d_ff:
        _, dgu, ddn = shared_mlp_bwd(dims, x, w_gate_up, w_down, dy, dx=dx, accumulate_dx=True)
        out.update(dw_gate_up=dgu, dw_down=ddn)
    return out


def _replace(d, **kw):
    import dataclasses
    return dataclasses.replace(d, **kw)


def expert_fwd_dense(dims: LayerDims, x, W, V, idx, gate, y_routed=None, ws=None):
    """The routed branch as two dense tcgen05 GEMMs (omnimoe_expert_fwd_dense)."""
    L = x.shape[0]
    lib = load()
    dc = dims.c()
    if y_routed is None:
        y_routed = torch.empty((L, dims.d), dtype=torch.float32, device=x.device)
    if ws is None:
        ws = torch.empty(max(lib.omnimoe_dense_workspace_size(ctypes.byref(dc), L), 1), dtype=torch.uint8,
                         device=x.device)
    _check(lib.omnimoe_expert_fwd_dense(ctypes.byref(dc), L, _ptr(x), _ptr(W), _ptr(V), _ptr(idx.contiguous()),
                                        _ptr(gate.contiguous()), _ptr(y_routed), _ptr(ws), ws.numel(), _stream()),
           "expert_fwd_dense")
    return y_routed


def layer_executor(dims: LayerDims, L: int) -> int:
    """The routed-branch executor (EXPERT_*) omnimoe_layer_fwd uses for L tokens."""
    dc = dims.c()
    return int(load().omnimoe_layer_executor(ctypes.byref(dc), L))


def expert_fwd_tokens(dims: LayerDims, x, W, V, idx, gate, y_routed=None, accumulate=False):
    """'w/o ECS' token-centric routed branch from the routing decision (omnimoe_expert_fwd_tokens)."""
    L = x.shape[0]
    hk = dims.n_heads * dims.top_k
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(idx, "idx", torch.int32, L * hk)
    _req(gate, "gate", torch.float32, L * hk)
    if y_routed is None:
        y_routed = torch.empty((L, dims.d), dtype=torch.float32, device=x.device)
        accumulate = False
    dc = dims.c()
    _check(load().omnimoe_expert_fwd_tokens(ctypes.byref(dc), L, _ptr(x), _ptr(W), _ptr(V), _ptr(idx), _ptr(gate),
                                            _ptr(y_routed), int(accumulate), _stream()), "expert_fwd_tokens")
    return y_routed


def pack_v(dims: LayerDims, V):
    """V [n][d] -> the SLICED layout [d/64][n][64] (include/omnimoe.h omnimoe_pack_v)."""
    n = V.numel() // dims.d
    _req(V, "V", dims.torch_dtype, n * dims.d)
    out = torch.empty((dims.d // 64, n, 64), dtype=V.dtype, device=V.device)
    dc = dims.c()
    _check(load().omnimoe_pack_v(ctypes.byref(dc), n, _ptr(V), _ptr(out), _stream()), "pack_v")
    return out


def expert_fwd(dims: LayerDims, x, W_loc, V_loc, plan, y_routed=None, accumulate=False, ws=None, passes=3):
    """passes: 3 = the whole routed branch; 1 / 2 = pass Z / pass V of the SLICED
    executor alone (measurement, omnimoe_expert_fwd_pass)."""
    L = x.shape[0]
    n_loc = plan["expert_end"] - plan["expert_begin"]
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(W_loc, "W_loc", dims.torch_dtype, n_loc * dims.d)
    _req(V_loc, "V_loc", dims.torch_dtype, n_loc * dims.d)
    if y_routed is None:
        y_routed = torch.empty((L, dims.d), dtype=torch.float32, device=x.device)
        accumulate = False
    _req(y_routed, "y_routed", torch.float32, L * dims.d)
    ws = ws if ws is not None else workspace(dims, L, WS_EXPERT, x.device)
    dc, cp = dims.c(), _cplan(plan)
    if passes == 3:
        _check(load().omnimoe_expert_fwd(ctypes.byref(dc), L, _ptr(x), _ptr(W_loc), _ptr(V_loc),
                                         ctypes.byref(cp), _ptr(y_routed), int(accumulate), _ptr(ws),
                                         ws.numel(), _stream()), "expert_fwd")
    else:
        _check(load().omnimoe_expert_fwd_pass(ctypes.byref(dc), L, _ptr(x), _ptr(W_loc), _ptr(V_loc),
                                              ctypes.byref(cp), _ptr(y_routed), int(accumulate), int(passes),
                                              _ptr(ws), ws.numel(), _stream()), "expert_fwd_pass")
    return y_routed


def shared_mlp(dims: LayerDims, x, w_gate_up, w_down, y_routed=None, y=None, ws=None):
    L = x.shape[0]
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(w_gate_up, "w_gate_up", dims.torch_dtype, 2 * dims.d_ff * dims.d)
    _req(w_down, "w_down", dims.torch_dtype, dims.d * dims.d_ff)
    if y_routed is not None:
        _req(y_routed, "y_routed", torch.float32, L * dims.d)
    y = y if y is not None else torch.empty((L, dims.d), dtype=dims.torch_dtype, device=x.device)
    ws = ws if ws is not None else workspace(dims, L, WS_MLP, x.device)
    dc = dims.c()
    _check(load().omnimoe_shared_mlp(ctypes.byref(dc), L, _ptr(x), _ptr(w_gate_up), _ptr(w_down),
                                     _ptr(y_routed), _ptr(y), _ptr(ws), ws.numel(), _stream()),
           "shared_mlp")
    return y


def layer_fwd(dims: LayerDims, x, subkeys, W, V, w_gate_up=None, w_down=None, y=None, ws=None,
              return_routing=False):
    L = x.shape[0]
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(subkeys, "subkeys", dims.torch_dtype, dims.n_heads * dims.router_rows * dims.d)
    _req(W, "W", dims.torch_dtype, dims.N * dims.d)
    _req(V, "V", dims.torch_dtype, dims.N * dims.d)
    if dims.d_ff:
        _req(w_gate_up, "w_gate_up", dims.torch_dtype, 2 * dims.d_ff * dims.d)
        _req(w_down, "w_down", dims.torch_dtype, dims.d * dims.d_ff)
    y = y if y is not None else torch.empty((L, dims.d), dtype=dims.torch_dtype, device=x.device)
    idx = gate = None
    if return_routing:
        idx = torch.empty((L, dims.n_heads, dims.top_k), dtype=torch.int32, device=x.device)
        gate = torch.empty((L, dims.n_heads, dims.top_k), dtype=torch.float32, device=x.device)
    ws = ws if ws is not None else workspace(dims, L, WS_LAYER, x.device)
    dc = dims.c()
    _check(load().omnimoe_layer_fwd(ctypes.byref(dc), L, _ptr(x), _ptr(subkeys), _ptr(W), _ptr(V),
                                    _ptr(w_gate_up), _ptr(w_down), _ptr(y), _ptr(idx), _ptr(gate),
                                    _ptr(ws), ws.numel(), _stream()), "layer_fwd")
    return (y, idx, gate) if return_routing else y


def layer_fwd_host(dims: LayerDims, x_host, subkeys, W, V, w_gate_up=None, w_down=None, y_host=None, x_dev=None,
                   y_dev=None, ws=None, chunks=4, copy_stream=None):
    """omnimoe_layer_fwd_host: x and y in (pinned) host memory, transfers overlapped with the
    router and the shared MLP.  Returns y_host; complete on the current stream."""
    L = x_host.shape[0]
    if x_host.is_cuda:
        raise OmniMoEError("x_host must be a host tensor")
    dev = torch.device("cuda", torch.cuda.current_device())
    x_dev = x_dev if x_dev is not None else torch.empty((L, dims.d), dtype=dims.torch_dtype, device=dev)
    y_dev = y_dev if y_dev is not None else torch.empty((L, dims.d), dtype=dims.torch_dtype, device=dev)
    y_host = y_host if y_host is not None else torch.empty((L, dims.d), dtype=dims.torch_dtype).pin_memory()
    copy_stream = copy_stream or torch.cuda.Stream()
    ws = ws if ws is not None else workspace(dims, L, WS_LAYER, dev)
    dc = dims.c()
    _check(load().omnimoe_layer_fwd_host(ctypes.byref(dc), L, ctypes.c_void_p(x_host.data_ptr()), _ptr(x_dev),
                                         _ptr(subkeys), _ptr(W), _ptr(V), _ptr(w_gate_up), _ptr(w_down), _ptr(y_dev),
                                         ctypes.c_void_p(y_host.data_ptr()), int(chunks), _ptr(ws), ws.numel(),
                                         _stream(), ctypes.c_void_p(copy_stream.cuda_stream)), "layer_fwd_host")
    return y_host


def router_logits(dims: LayerDims, x, subkeys, method=LOGITS_ROUTE, ws=None):
    """Sub-key logits [L][h][N_r+N_c] fp32.  method: LOGITS_ROUTE (what route uses),
    LOGITS_EXACT_F64, LOGITS_BF16_FAST (inexact fp32-accumulated tcgen05, measurement only)."""
    L = x.shape[0]
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(subkeys, "subkeys", dims.torch_dtype, dims.n_heads * dims.router_rows * dims.d)
    out = torch.empty((L, dims.n_heads, dims.router_rows), dtype=torch.float32, device=x.device)
    ws = ws if ws is not None else workspace(dims, L, WS_ROUTE, x.device)
    dc = dims.c()
    _check(load().omnimoe_router_logits(ctypes.byref(dc), L, _ptr(x), _ptr(subkeys), _ptr(out), int(method),
                                        _ptr(ws), ws.numel(), _stream()), "router_logits")
    return out


def gemm_bf16(A, B):
    M, K = A.shape
    N = B.shape[0]
    _req(A, "A", torch.bfloat16)
    _req(B, "B", torch.bfloat16)
    C = torch.empty((M, N), dtype=torch.float32, device=A.device)
    _check(load().omnimoe_gemm_bf16(M, N, K, _ptr(A), _ptr(B), _ptr(C), _stream()), "gemm_bf16")
    return C


# ---------------------------------------------------------------- expert parallelism
def ep_pack(dims: LayerDims, x, idx, gate, R: int):
    """Dispatch buffers for R expert shards (include/omnimoe.h omnimoe_ep_pack).
    Returns (x_send, rec_send, inv, counts) with counts a device int64 [R][2] tensor
    (rows, records per destination); x_send / rec_send are capacity-sized (R*L rows,
    L*h*K records): the first sum of each column of counts are valid."""
    L = x.shape[0]
    hk = dims.n_heads * dims.top_k
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(idx, "idx", torch.int32, L * hk)
    _req(gate, "gate", torch.float32, L * hk)
    x_send = torch.empty((max(R * L, 1), dims.d), dtype=dims.torch_dtype, device=x.device)
    rec = torch.empty((max(L * hk, 1), 3), dtype=torch.int32, device=x.device)
    inv = torch.empty((R, max(L, 1)), dtype=torch.int32, device=x.device)
    off = torch.empty(2 * R + 2, dtype=torch.int32, device=x.device)
    counts = torch.empty((R, 2), dtype=torch.int64, device=x.device)
    nb = ctypes.c_size_t(0)
    _check(load().omnimoe_ep_pack_workspace_size(L, R, ctypes.byref(nb)), "ep_pack_workspace_size")
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=x.device)
    dc = dims.c()
    _check(load().omnimoe_ep_pack(ctypes.byref(dc), L, R, _ptr(x), _ptr(idx), _ptr(gate), _ptr(x_send), _ptr(rec),
                                  _ptr(inv), _ptr(off), _ptr(counts), _ptr(ws), ws.numel(), _stream()), "ep_pack")
    return x_send, rec, inv[:, :L], counts


def ep_partials(dims: LayerDims, y_part):
    """fp32 partial rows -> bf16 for the return all-to-all (omnimoe_ep_partials)."""
    rows = y_part.shape[0]
    _req(y_part, "y_part", torch.float32, rows * dims.d)
    out = torch.empty((rows, dims.d), dtype=torch.bfloat16, device=y_part.device)
    dc = dims.c()
    _check(load().omnimoe_ep_partials(rows, ctypes.byref(dc), _ptr(y_part), _ptr(out), _stream()), "ep_partials")
    return out


def ep_unpack(rec, R: int, task_off, tok_off):
    """Received records -> (ids, gate, token) task arrays over the local expert range."""
    M = rec.shape[0]
    _req(rec, "rec", torch.int32, M * 3)
    _req(task_off, "task_off", torch.int64, R + 1)
    _req(tok_off, "tok_off", torch.int64, R + 1)
    ids = torch.empty(max(M, 1), dtype=torch.int32, device=rec.device)
    gate = torch.empty(max(M, 1), dtype=torch.float32, device=rec.device)
    tok = torch.empty(max(M, 1), dtype=torch.int32, device=rec.device)
    _check(load().omnimoe_ep_unpack(M, R, _ptr(rec), _ptr(task_off), _ptr(tok_off), _ptr(ids), _ptr(gate),
                                    _ptr(tok), _stream()), "ep_unpack")
    return ids[:M], gate[:M], tok[:M]


def ep_combine(dims: LayerDims, y_ret, inv, tok_off, L: int):
    """y_routed[l] = sum_s y_ret[tok_off[s] + inv[s][l]] in rank order (fp32 accumulation;
    y_ret bf16 from ep_partials, or fp32)."""
    R = inv.shape[0]
    _req(inv, "inv", torch.int32, R * L)
    _req(tok_off, "tok_off", torch.int64, R + 1)
    bf = y_ret.dtype == torch.bfloat16
    if y_ret.numel():
        _req(y_ret, "y_ret", torch.bfloat16 if bf else torch.float32)
    y = torch.empty((L, dims.d), dtype=torch.float32, device=inv.device)
    dc = dims.c()
    _check(load().omnimoe_ep_combine(ctypes.byref(dc), L, R, _ptr(y_ret) if y_ret.numel() else None, int(bf),
                                     _ptr(inv), _ptr(tok_off), _ptr(y), _stream()), "ep_combine")
    return y


def shared_mlp_hidden(dims: LayerDims, x, w_gate_up, H=None):
    """Shared-MLP GEMM-1 into an opaque H buffer (omnimoe_shared_mlp_hidden)."""
    L = x.shape[0]
    _req(x, "x", dims.torch_dtype, L * dims.d)
    _req(w_gate_up, "w_gate_up", dims.torch_dtype, 2 * dims.d_ff * dims.d)
    H = H if H is not None else workspace(dims, L, WS_MLP, x.device)
    dc = dims.c()
    _check(load().omnimoe_shared_mlp_hidden(ctypes.byref(dc), L, _ptr(x), _ptr(w_gate_up), _ptr(H), H.numel(),
                                            _stream()), "shared_mlp_hidden")
    return H


def shared_mlp_out(dims: LayerDims, L: int, H, w_down, y_routed=None, y=None):
    """Shared-MLP GEMM-2 + combine: y = H W_down^T + y_routed (omnimoe_shared_mlp_out)."""
    _req(w_down, "w_down", dims.torch_dtype, dims.d * dims.d_ff)
    if y_routed is not None:
        _req(y_routed, "y_routed", torch.float32, L * dims.d)
    y = y if y is not None else torch.empty((L, dims.d), dtype=dims.torch_dtype, device=H.device)
    dc = dims.c()
    _check(load().omnimoe_shared_mlp_out(ctypes.byref(dc), L, _ptr(H), H.numel(), _ptr(w_down), _ptr(y_routed),
                                         _ptr(y), _stream()), "shared_mlp_out")
    return y
