"""Builds the seeded synthetic inputs of a workload (shapes and scale
exponents only -- no arithmetic of the method).  Device tensors come from
synth/libsynth.so; the host side regenerates any rows it needs with the numpy
twin (synth.gen_rows_*), bit-identically."""
from __future__ import annotations

import torch

from . import (NORMAL, TID_SUBKEYS, TID_V, TID_W, TID_W_DOWN, TID_W_GATE_UP, TID_X,
               default_exponents)
from .cuda import make


def tensor_specs(dims, L):
    """(name, tensor id, shape) of every input of the layer."""
    N = dims.n_rows * dims.n_cols
    R = N if getattr(dims, "router", 0) == 2 else dims.n_rows + dims.n_cols  # dense-router ablation: N gate rows
    specs = [("x", TID_X, (L, dims.d)), ("subkeys", TID_SUBKEYS, (dims.n_heads, R, dims.d)),
             ("W", TID_W, (N, dims.d)), ("V", TID_V, (N, dims.d))]
    if dims.d_ff:
        specs += [("w_gate_up", TID_W_GATE_UP, (2 * dims.d_ff, dims.d)),
                  ("w_down", TID_W_DOWN, (dims.d, dims.d_ff))]
    return specs


def make_inputs(dims, L, seed, mode=NORMAL, device="cuda", skip=(), token_begin=0, expert_rows=None):
    """Inputs of the layer.  token_begin: the batch is tokens [token_begin,
    token_begin + L) of the global stream; expert_rows=(begin, end): only these
    rows of W and V (an expert-parallel shard), identical to the same rows of
    the full tables."""
    ex = default_exponents(dims.d, dims.d_ff, mode)
    dt = torch.bfloat16 if dims.dtype == 0 else torch.float32
    out = {"exponents": ex, "seed": seed, "mode": mode}
    for name, tid, shape in tensor_specs(dims, L):
        if name in skip:
            continue
        base = 0
        if name == "x":
            base = token_begin * dims.d
        elif name in ("W", "V") and expert_rows is not None:
            base = expert_rows[0] * dims.d
            shape = (expert_rows[1] - expert_rows[0], dims.d)
        out[name] = make(shape, dt, seed, tid, ex[tid], mode, device, base)
    return out
