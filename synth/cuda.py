"""ctypes binding of synth/libsynth.so: fills CUDA tensors with the seeded
generator of synth/__init__.py, bit-identically, directly in HBM."""
from __future__ import annotations

import ctypes
import os

import torch

from . import NORMAL

_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise RuntimeError(f"{_SO} not built (run __graft_entry__.build())")
        _lib = ctypes.CDLL(_SO)
        _lib.synth_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        _lib.synth_fill.restype = ctypes.c_int
    return _lib


def fill_(t: torch.Tensor, seed: int, tensor_id: int, e: int, mode: int = NORMAL, base: int = 0) -> torch.Tensor:
    """Fill t with draws base .. base + numel - 1 of (seed, tensor_id)."""
    assert t.is_cuda and t.is_contiguous() and t.dtype in (torch.bfloat16, torch.float32)
    rc = _load().synth_fill(seed, tensor_id, base, t.numel(), e, mode, int(t.dtype == torch.bfloat16),
                            ctypes.c_void_p(t.data_ptr()),
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_fill failed with cuda error {rc}")
    return t


def make(shape, dtype, seed, tensor_id, e, mode=NORMAL, device="cuda", base=0):
    return fill_(torch.empty(shape, dtype=dtype, device=device), seed, tensor_id, e, mode, base)
