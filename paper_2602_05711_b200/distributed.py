"""Expert-parallel OmniMoE layer forward over R ranks.

Tokens are data-parallel (L_loc per rank); the atomic-expert tables W, V are
row-sharded: rank r owns flat ids [r*N/R, (r+1)*N/R), i.e. whole grid rows
(n = i*N_c + j, reading Q6).  The sub-key tables and the shared MLP are
replicated.  One forward, per rank:

  1. route the local tokens (omnimoe_route: exact, batch-independent, so ids are
     bit-identical to a single-GPU run) and pack the dispatch buffers
     (omnimoe_ep_pack: each token once per destination + one record per task);
  2. all-to-all of the per-destination counts, then of the x rows and records
     (NCCL all_to_all_single over NVLink / NVSwitch);
  3. unpack (omnimoe_ep_unpack), schedule + grouped expert compute on the local
     shard (omnimoe_schedule + omnimoe_expert_fwd over the received rows);
  4. all-to-all of the partial y rows back to the home ranks;
  5. combine in fixed rank order (omnimoe_ep_combine) and add the shared MLP
     (omnimoe_shared_mlp, bf16 output).

The exchange is written against a small communicator interface so the same
phases run over torch.distributed (NCCL on B200, gloo in the CPU tests) and
over an in-process loopback of R virtual ranks on one GPU.  Which kernels run
is also pluggable (``ops``): the product uses ``LibOps`` (libomnimoe.so); the
CPU tests inject the oracle -- there is no CPU path in the product.
"""
from __future__ import annotations

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

    def route(self, x, subkeys):
        idx, gate, _ = om.route(self.dims, x, subkeys, want_score=False)
        hk = self.dims.n_heads * self.dims.top_k
        return idx.reshape(-1, hk), gate.reshape(-1, hk)

    def pack(self, x, idx, gate, R):
        return om.ep_pack(self.dims, x, idx.contiguous(), gate.contiguous(), R)

    def unpack(self, rec, R, task_off, tok_off):
        return om.ep_unpack(rec, R, task_off, tok_off)

    def expert(self, x_recv, W_loc, V_loc, ids, gate, tok, n_loc):
        """V_loc is [n_loc][d], or [d/64][n_loc][64] when dims.v_layout is V_SLICED
        (om.pack_v of the shard); the SLICED executor writes every row of y."""
        sliced = self.dims.v_layout == om.V_SLICED
        rows = x_recv.shape[0]
        if ids.numel() == 0 or rows == 0:
            return torch.zeros((rows, self.dims.d), dtype=torch.float32, device=x_recv.device)
        y = (torch.empty if sliced else torch.zeros)((rows, self.dims.d), dtype=torch.float32, device=x_recv.device)
        plan = om.schedule(self.dims, ids, gate, token=tok, expert_begin=0, expert_end=n_loc, n_tokens=rows)
        return om.expert_fwd(self.dims, x_recv, W_loc, V_loc, plan, y_routed=y, accumulate=not sliced)

    def combine(self, y_ret, inv, tok_off, L):
        return om.ep_combine(self.dims, y_ret, inv, tok_off, L)

    def mlp(self, x, y_routed):
        if self.dims.d_ff:
            return om.shared_mlp(self.dims, x, self._wgu, self._wdn, y_routed=y_routed)
        return y_routed.to(self.dims.torch_dtype)

    def set_mlp(self, w_gate_up, w_down):
        self._wgu, self._wdn = w_gate_up, w_down


# ---------------------------------------------------------------- communicators
class TorchComm:
    """all_to_all over a torch.distributed process group (NCCL or gloo)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange_counts(self, counts: List[int], device) -> List[int]:
        t = torch.tensor(counts, dtype=torch.int64, device=device)
        out = torch.empty_like(t)
        dist.all_to_all_single(out, t, group=self.group)
        return out.cpu().tolist()

    def exchange(self, send, send_splits, recv_splits):
        out = torch.empty((sum(recv_splits),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(out, send.contiguous(), output_split_sizes=recv_splits,
                               input_split_sizes=send_splits, group=self.group)
        return out


# ---------------------------------------------------------------- per-rank state
@dataclass
class RankState:
    x: torch.Tensor                    # [L_loc][d] local tokens
    W_loc: torch.Tensor                # [N/R][d]
    V_loc: torch.Tensor
    L: int = 0
    inv: Optional[torch.Tensor] = None
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
    st.x_send, st.rec_send, st.inv, offs = ops.pack(st.x, idx, gate, R)
    st.send_tok = [offs[s + 1] - offs[s] for s in range(R)]
    st.send_task = [offs[R + 2 + s] - offs[R + 1 + s] for s in range(R)]


def phase_expert(ops, st: RankState, R: int, n_loc: int):
    """Unpack the received records and run schedule + expert compute on the shard."""
    dev = st.x_recv.device
    ids, gate, tok = ops.unpack(st.rec_recv.contiguous(), R, _offsets(st.recv_task, dev), _offsets(st.recv_tok, dev))
    st.y_part = ops.expert(st.x_recv.contiguous(), st.W_loc, st.V_loc, ids, gate, tok, n_loc)


def phase_combine(ops, st: RankState):
    """Add the returned partial rows in rank order, then the shared MLP (a7 + a8)."""
    y_routed = ops.combine(st.y_ret.contiguous(), st.inv.contiguous(), _offsets(st.send_tok, st.x.device), st.L)
    st.y = ops.mlp(st.x, y_routed)


# ---------------------------------------------------------------- drivers
def ep_layer_fwd(ops, comm: TorchComm, x_loc, subkeys, W_loc, V_loc, n_per: int, marks=None):
    """One expert-parallel layer forward on this rank (torch.distributed).
    marks: optional callable(name) invoked between phases (bench timing)."""
    mark = marks or (lambda name: None)
    R = comm.world
    st = RankState(x=x_loc, W_loc=W_loc, V_loc=V_loc)
    mark("start")
    phase_dispatch(ops, st, subkeys, R)
    mark("dispatch")
    pairs = [v for s in range(R) for v in (st.send_tok[s], st.send_task[s])]  # block s -> rank s
    st.recv_tok, st.recv_task = _split_counts(comm.exchange_counts(pairs, x_loc.device), R)
    st.x_recv = comm.exchange(st.x_send, st.send_tok, st.recv_tok)
    st.rec_recv = comm.exchange(st.rec_send, st.send_task, st.recv_task)
    mark("all_to_all_dispatch")
    phase_expert(ops, st, R, n_per)
    mark("expert")
    st.y_ret = comm.exchange(st.y_part, st.recv_tok, st.send_tok)
    mark("all_to_all_combine")
    phase_combine(ops, st)
    mark("combine_mlp")
    return st.y


def _split_counts(received, R):
    """The counts travel as pairs (rows, records): element block s of the send
    tensor goes to rank s, and ``received`` is the concatenation of the pairs
    from every source rank."""
    return [received[2 * s] for s in range(R)], [received[2 * s + 1] for s in range(R)]


def ep_layer_fwd_loopback(ops, xs, subkeys, W_locs, V_locs, n_per: int):
    """R virtual ranks in one process (one GPU): the same phases, with the
    all-to-alls done as slices and concatenations."""
    R = len(xs)
    sts = [RankState(x=xs[r], W_loc=W_locs[r], V_loc=V_locs[r]) for r in range(R)]
    for st in sts:
        phase_dispatch(ops, st, subkeys, R)

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
        phase_combine(ops, st)
    return [st.y for st in sts]


def shard_rows(t, R: int, r: int):
    n = t.shape[0] // R
    return t[r * n:(r + 1) * n]
