"""Expert-parallel OmniMoE layer forward over R ranks.

Tokens are data-parallel (L_loc per rank); the atomic-expert tables W, V are
row-sharded: rank r owns flat ids [r*N/R, (r+1)*N/R), i.e. whole grid rows
(n = i*N_c + j, reading Q6).  The sub-key tables and the shared MLP are
replicated.  One forward, per rank:

  1. route the local tokens (omnimoe_route: exact, batch-independent, so ids are
     bit-identical to a single-GPU run) and pack the dispatch buffers
     (omnimoe_ep_pack: each token once per destination + one record per task, and
     the per-destination counts on the device);
  2. all-to-all of the counts (device to device; ONE host read of the send and
     receive counts per forward sizes the exchanges), then of the x rows and the
     records (NCCL all_to_all_single over NVLink / NVSwitch); the shared MLP's
     first GEMM (it needs x only) runs meanwhile on a side stream;
  3. unpack (omnimoe_ep_unpack), schedule + grouped expert compute on the local
     shard (omnimoe_schedule + omnimoe_expert_fwd over the received rows);
  4. all-to-all of the partial y rows back to the home ranks, in bf16
     (omnimoe_ep_partials: half the bytes of fp32);
  5. combine in fixed rank order with fp32 accumulation (omnimoe_ep_combine) and
     the shared MLP's second GEMM + combine (omnimoe_shared_mlp_out, bf16 output).

The exchange is written against a small communicator interface so the same
phases run over torch.distributed (NCCL on B200, gloo in the CPU tests) and
over an in-process loopback of R virtual ranks on one GPU.  Which kernels run
is also pluggable (``ops``): the product uses ``LibOps`` (libomnimoe.so); the
CPU tests inject the oracle -- there is no CPU path in the product.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import List, Optional

import torch
import torch.distributed as dist

from . import omnimoe as om


# ---------------------------------------------------------------- kernels
class LibOps:
    """The product's kernels (C ABI of libomnimoe.so)."""

    def __init__(self, dims: om.LayerDims):
        self.dims = dims
        # the layer's routing: candidate order (same ids and gates as key order; the
        # schedule re-sorts the tasks anyway)
        self._rdims = dataclasses.replace(dims, route_order=om.ORDER_CANDIDATE)
        self.last_route = None

    def route(self, x, subkeys):
        idx, gate, _ = om.route(self._rdims, x, subkeys, want_score=False)
        hk = self.dims.n_heads * self.dims.top_k
        self.last_route = (idx.reshape(-1, hk), gate.reshape(-1, hk))
        return self.last_route

    def pack(self, x, idx, gate, R):
        return om.ep_pack(self.dims, x, idx.contiguous(), gate.contiguous(), R)

    def unpack(self, rec, R, task_off, tok_off):
        return om.ep_unpack(rec, R, task_off, tok_off)

    def expert(self, x_recv, W_loc, V_loc, ids, gate, tok, n_loc):
        """V_loc is [n_loc][d], or [d/64][n_loc][64] when dims.v_layout is V_SLICED
        (om.pack_v of the shard); the SLICED executor writes every row of y.  Returns
        the partial rows in bf16 (the return trip's payload)."""
        sliced = self.dims.v_layout == om.V_SLICED
        rows = x_recv.shape[0]
        if ids.numel() == 0 or rows == 0:
            return torch.zeros((rows, self.dims.d), dtype=torch.bfloat16, device=x_recv.device)
        y = (torch.empty if sliced else torch.zeros)((rows, self.dims.d), dtype=torch.float32, device=x_recv.device)
        plan = om.schedule(self.dims, ids, gate, token=tok, expert_begin=0, expert_end=n_loc, n_tokens=rows)
        # the partials go back in bf16, so pass V may take the activations in bf16 as
        # omnimoe_layer_fwd does (reading Q21)
        ed = dataclasses.replace(self.dims, flags=self.dims.flags | om.FLAG_ACT_BF16)
        y = om.expert_fwd(ed, x_recv, W_loc, V_loc, plan, y_routed=y, accumulate=not sliced)
        return om.ep_partials(self.dims, y)

    def combine(self, y_ret, inv, tok_off, L):
        return om.ep_combine(self.dims, y_ret, inv, tok_off, L)

    def mlp_hidden(self, x):
        return om.shared_mlp_hidden(self.dims, x, self._wgu) if self.dims.d_ff else None

    def mlp_out(self, x, H, y_routed):
        if self.dims.d_ff:
            return om.shared_mlp_out(self.dims, x.shape[0], H, self._wdn, y_routed=y_routed)
        return y_routed.to(self.dims.torch_dtype)

    def set_mlp(self, w_gate_up, w_down):
        self._wgu, self._wdn = w_gate_up, w_down


# ---------------------------------------------------------------- communicators
class TorchComm:
    """all_to_all over a torch.distributed process group: NCCL (device to device), or
    gloo -- with CPU tensors as they are, with CUDA tensors staged through host memory
    (the CPU tests, and the 2-process dry run on one GPU)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = dist.get_backend(group) == "gloo"

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        if self.staged and inp.is_cuda:
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), output_split_sizes=out_splits, input_split_sizes=in_splits,
                                   group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                   group=self.group)
        return out

    def exchange_counts(self, counts):
        """counts: int64 [R][2] (rows, records) for each destination -> the same for each
        source, as host lists (sent, received): the forward's one host synchronisation."""
        recv = self._a2a(torch.empty_like(counts), counts.contiguous())
        both = torch.stack([counts, recv]).cpu()
        return both[0].tolist(), both[1].tolist()

    def exchange(self, send, send_splits, recv_splits):
        out = torch.empty((sum(recv_splits),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        return self._a2a(out, send[:sum(send_splits)].contiguous(), recv_splits, send_splits)


# ---------------------------------------------------------------- per-rank state
@dataclass
class RankState:
    x: torch.Tensor                    # [L_loc][d] local tokens
    W_loc: torch.Tensor                # [N/R][d]
    V_loc: torch.Tensor
    L: int = 0
    inv: Optional[torch.Tensor] = None
    counts: Optional[torch.Tensor] = None              # int64 [R][2] (rows, records) per destination
    send_tok: List[int] = field(default_factory=list)    # rows sent to each rank
    send_task: List[int] = field(default_factory=list)   # records sent to each rank
    x_send: Optional[torch.Tensor] = None
    rec_send: Optional[torch.Tensor] = None
    recv_tok: List[int] = field(default_factory=list)
    recv_task: List[int] = field(default_factory=list)
    x_recv: Optional[torch.Tensor] = None
    rec_recv: Optional[torch.Tensor] = None
    y_part: Optional[torch.Tensor] = None
    y_ret: Optional[torch.Tensor] = None
    y: Optional[torch.Tensor] = None


def _offsets(counts, device):
    off = [0]
    for c in counts:
        off.append(off[-1] + c)
    return torch.tensor(off, dtype=torch.int64, device=device)


def phase_dispatch(ops, st: RankState, subkeys, R: int):
    """Route the local tokens and pack one message per destination rank."""
    st.L = st.x.shape[0]
    idx, gate = ops.route(st.x, subkeys)
    st.x_send, st.rec_send, st.inv, st.counts = ops.pack(st.x, idx, gate, R)


def phase_expert(ops, st: RankState, R: int, n_loc: int):
    """Unpack the received records and run schedule + expert compute on the shard."""
    dev = st.x_recv.device
    ids, gate, tok = ops.unpack(st.rec_recv.contiguous(), R, _offsets(st.recv_task, dev), _offsets(st.recv_tok, dev))
    st.y_part = ops.expert(st.x_recv.contiguous(), st.W_loc, st.V_loc, ids, gate, tok, n_loc)


def phase_combine(ops, st: RankState, H):
    """Add the returned partial rows in rank order, then the shared MLP's second GEMM
    (a7 + a8)."""
    y_routed = ops.combine(st.y_ret.contiguous(), st.inv.contiguous(), _offsets(st.send_tok, st.x.device), st.L)
    st.y = ops.mlp_out(st.x, H, y_routed)


class _Side:
    """The shared MLP's first GEMM on a side stream (CUDA), joined before its second."""

    def __init__(self, x):
        self.cuda = x.is_cuda
        if self.cuda:
            self.stream = torch.cuda.Stream(device=x.device)
            self.stream.wait_stream(torch.cuda.current_stream(x.device))

    def run(self, fn, *args):
        if not self.cuda:
            return fn(*args)
        with torch.cuda.stream(self.stream):
            out = fn(*args)
        self.event = torch.cuda.Event()
        self.event.record(self.stream)
        return out

    def join(self, x, *tensors):
        if self.cuda:
            torch.cuda.current_stream(x.device).wait_event(self.event)
            for t in tensors:  # allocated on the side stream, consumed on the main one
                if t is not None:
                    t.record_stream(torch.cuda.current_stream(x.device))


# ---------------------------------------------------------------- drivers
def ep_layer_fwd(ops, comm: TorchComm, x_loc, subkeys, W_loc, V_loc, n_per: int, marks=None, return_state=False):
    """One expert-parallel layer forward on this rank (torch.distributed).
    marks: optional callable(name) invoked between phases (bench timing);
    return_state: also return the RankState (message sizes, for the bench)."""
    mark = marks or (lambda name: None)
    R = comm.world
    st = RankState(x=x_loc, W_loc=W_loc, V_loc=V_loc)
    mark("start")
    phase_dispatch(ops, st, subkeys, R)
    side = _Side(x_loc)
    H = side.run(ops.mlp_hidden, x_loc)  # overlaps the exchanges below
    mark("dispatch")
    sent, recv = comm.exchange_counts(st.counts)
    st.send_tok, st.send_task = [c[0] for c in sent], [c[1] for c in sent]
    st.recv_tok, st.recv_task = [c[0] for c in recv], [c[1] for c in recv]
    st.x_recv = comm.exchange(st.x_send, st.send_tok, st.recv_tok)
    st.rec_recv = comm.exchange(st.rec_send, st.send_task, st.recv_task)
    mark("all_to_all_dispatch")
    phase_expert(ops, st, R, n_per)
    mark("expert")
    st.y_ret = comm.exchange(st.y_part, st.recv_tok, st.send_tok)
    mark("all_to_all_combine")
    side.join(x_loc, H)
    phase_combine(ops, st, H)
    mark("combine_mlp")
    return (st.y, st) if return_state else st.y


def ep_layer_fwd_loopback(ops, xs, subkeys, W_locs, V_locs, n_per: int):
    """R virtual ranks in one process (one GPU): the same phases, with the
    all-to-alls done as slices and concatenations."""
    R = len(xs)
    sts = [RankState(x=xs[r], W_loc=W_locs[r], V_loc=V_locs[r]) for r in range(R)]
    for st in sts:
        phase_dispatch(ops, st, subkeys, R)
        sent = st.counts.cpu().tolist()
        st.send_tok, st.send_task = [c[0] for c in sent], [c[1] for c in sent]

    def blocks(t, counts):
        out, o = [], 0
        for c in counts:
            out.append(t[o:o + c])
            o += c
        return out

    for r, st in enumerate(sts):
        st.recv_tok = [sts[s].send_tok[r] for s in range(R)]
        st.recv_task = [sts[s].send_task[r] for s in range(R)]
        st.x_recv = torch.cat([blocks(sts[s].x_send, sts[s].send_tok)[r] for s in range(R)])
        st.rec_recv = torch.cat([blocks(sts[s].rec_send, sts[s].send_task)[r] for s in range(R)])
    for st in sts:
        phase_expert(ops, st, R, n_per)
    for r, st in enumerate(sts):
        st.y_ret = torch.cat([blocks(sts[s].y_part, sts[s].recv_tok)[r] for s in range(R)])
    for st in sts:
        phase_combine(ops, st, ops.mlp_hidden(st.x))
    return [st.y for st in sts]


def shard_rows(t, R: int, r: int):
    n = t.shape[0] // R
    return t[r * n:(r + 1) * n]


# ---------------------------------------------------------------- fused device-API exchange (N3)
class _DevPtr:
    """A device buffer exposed to torch.as_tensor through __cuda_array_interface__."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class DevExchange:
    """The dispatch / return exchange on the NCCL device API (libomnimoe_ep.so,
    include/omnimoe_ep.h): symmetric windows, peer stores over NVLink from the GPU's own
    kernels, in-kernel LSA barriers -- no NCCL collective in the forward.  row_cap / rec_cap:
    capacities of the receive windows (rows and task records any rank can receive)."""

    def __init__(self, dims: om.LayerDims, row_cap: int, rec_cap: int, group=None):
        import ctypes
        import os
        from . import build
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libomnimoe_ep.so")
        if not os.path.exists(path):
            raise om.OmniMoEError(f"{path} not built (build.build_ep())")
        self.lib = lib = ctypes.CDLL(path)
        V, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        lib.omnimoe_ep_dev_unique_id_bytes.restype = ctypes.c_size_t
        lib.omnimoe_ep_dev_unique_id.argtypes = [V]
        lib.omnimoe_ep_dev_create.argtypes = [V, I32, I32, I64, I64, I64, ctypes.POINTER(V)]
        lib.omnimoe_ep_dev_destroy.argtypes = [V]
        lib.omnimoe_ep_dev_buffers.argtypes = [V, ctypes.POINTER(V), ctypes.POINTER(V), ctypes.POINTER(V),
                                               ctypes.POINTER(V)]
        lib.omnimoe_ep_dev_dispatch.argtypes = [V, V, V, V, V]
        lib.omnimoe_ep_dev_return.argtypes = [V, V, I64, V]
        lib.omnimoe_ep_last_error.restype = ctypes.c_char_p
        for f in ("omnimoe_ep_dev_unique_id", "omnimoe_ep_dev_create", "omnimoe_ep_dev_destroy",
                  "omnimoe_ep_dev_buffers", "omnimoe_ep_dev_dispatch", "omnimoe_ep_dev_return"):
            getattr(lib, f).restype = ctypes.c_int
        self.dims, self.row_cap, self.rec_cap = dims, row_cap, rec_cap
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        nb = lib.omnimoe_ep_dev_unique_id_bytes()
        uid = (ctypes.c_uint8 * nb)()
        if self.rank == 0:
            self._check(lib.omnimoe_ep_dev_unique_id(ctypes.cast(uid, V)), "unique_id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        ctypes.memmove(uid, box[0], nb)
        self.handle = V()
        self._check(lib.omnimoe_ep_dev_create(ctypes.cast(uid, V), self.rank, self.world, dims.d, row_cap, rec_cap,
                                              ctypes.byref(self.handle)), "create")
        px, pr, py, pc = V(), V(), V(), V()
        self._check(lib.omnimoe_ep_dev_buffers(self.handle, ctypes.byref(px), ctypes.byref(pr), ctypes.byref(py),
                                               ctypes.byref(pc)), "buffers")
        R = self.world
        self.x_recv = torch.as_tensor(_DevPtr(px.value, (row_cap, dims.d), "<i2"), device="cuda").view(torch.bfloat16)
        self.rec = torch.as_tensor(_DevPtr(pr.value, (rec_cap, 3), "<i4"), device="cuda")
        self.y_ret = torch.as_tensor(_DevPtr(py.value, (row_cap, dims.d), "<i2"), device="cuda").view(torch.bfloat16)
        self.counts = torch.as_tensor(_DevPtr(pc.value, (R, R, 2), "<i8"), device="cuda")

    def _check(self, rc, what):
        if rc != 0:
            raise om.OmniMoEError(f"ep_dev {what}: status {rc}: {self.lib.omnimoe_ep_last_error().decode()}")

    def _stream(self):
        import ctypes
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def dispatch(self, x_send, rec_send, counts):
        import ctypes
        self._check(self.lib.omnimoe_ep_dev_dispatch(self.handle, ctypes.c_void_p(x_send.data_ptr()),
                                                     ctypes.c_void_p(rec_send.data_ptr()),
                                                     ctypes.c_void_p(counts.contiguous().data_ptr()),
                                                     self._stream()), "dispatch")

    def return_(self, y_part):
        import ctypes
        self._check(self.lib.omnimoe_ep_dev_return(self.handle, ctypes.c_void_p(y_part.data_ptr()),
                                                   y_part.shape[0], self._stream()), "return")

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.omnimoe_ep_dev_destroy(self.handle)
            self.handle = None


def ep_layer_fwd_dev(ops: LibOps, dx: DevExchange, x_loc, subkeys, W_loc, V_loc, n_per: int, marks=None):
    """One expert-parallel layer forward with the fused device-API exchange (N3): same
    pack / unpack / schedule / expert / combine kernels as ep_layer_fwd, the messages moved by
    the GPU's own peer stores into the symmetric windows.  One 8 R^2-byte read of the counts
    matrix per forward sizes the receiver's schedule (its sizes are host values)."""
    mark = marks or (lambda name: None)
    R = dx.world
    st = RankState(x=x_loc, W_loc=W_loc, V_loc=V_loc)
    mark("start")
    phase_dispatch(ops, st, subkeys, R)
    side = _Side(x_loc)
    H = side.run(ops.mlp_hidden, x_loc)
    mark("dispatch")
    dx.dispatch(st.x_send, st.rec_send, st.counts)
    cm = dx.counts.cpu()  # [src][dst][rows, records]
    me = dx.rank
    rows = int(cm[:, me, 0].sum())
    M = int(cm[:, me, 1].sum())
    st.send_tok = cm[me, :, 0].tolist()
    if rows > dx.row_cap or M > dx.rec_cap or sum(st.send_tok) > dx.row_cap:
        raise om.OmniMoEError(f"ep_dev: capacities exceeded (rows {rows}, records {M}, caps {dx.row_cap}, {dx.rec_cap})")
    mark("all_to_all_dispatch")
    dev = x_loc.device
    z = torch.zeros(2, dtype=torch.int64, device=dev)
    ids, gate, tok = ops.unpack(dx.rec[:M], 1, torch.tensor([0, M], dtype=torch.int64, device=dev), z)
    st.y_part = ops.expert(dx.x_recv[:rows], W_loc, V_loc, ids, gate, tok, n_per)
    mark("expert")
    dx.return_(st.y_part)
    st.y_ret = dx.y_ret[:sum(st.send_tok)]
    mark("all_to_all_combine")
    side.join(x_loc, H)
    phase_combine(ops, st, H)
    mark("combine_mlp")
    return st.y
