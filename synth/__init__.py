"""Seeded synthetic-input generator shared by the oracle harness and the GPU path.

This module holds NO arithmetic of the OmniMoE method: it only turns
(seed, tensor id, element index) into a number.  Both sides of the parity
tests draw their inputs from it -- the host implementation below (numpy), and
the bit-identical device implementation in ``synth/synth.cu`` (built into
``synth/libsynth.so``) which the bench uses to fill multi-GB expert tables
directly in HBM.  A GPU test checks host/device bit identity.

Generator (SURVEY.md 8(d) "Synthetic inputs"):

    key  = (seed << 56) ^ (tensor_id << 48) ^ index          (index < 2**48)
    h    = splitmix64(key)
    mode NORMAL: v = sum of the four 16-bit fields of h - 131070
                 (integer in [-131070, 131070], std ~= 37837, ~Gaussian)
                 value = v * 2**-e   (exact in fp32; bf16 tensors round it
                                      to nearest-even)
    mode DYADIC: v = (h mod 9) - 4, value = v * 2**-e
                 (x uses e = 2, sub-keys / W use e = 6: SURVEY.md P6)

Tensor ids: X=1, SUBKEYS=2, W=3, V=4, W_GATE_UP=5, W_DOWN=6.
"""
from __future__ import annotations

import math
import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

TID_X, TID_SUBKEYS, TID_W, TID_V, TID_W_GATE_UP, TID_W_DOWN = 1, 2, 3, 4, 5, 6

NORMAL, DYADIC = 0, 1
INT_STD = math.sqrt(4 * (65536.0 ** 2 - 1) / 12.0)  # std of the 4x16-bit sum


def scale_exponent(target_std: float) -> int:
    """e such that INT_STD * 2**-e is the power-of-two scaling nearest target_std."""
    return int(round(math.log2(INT_STD / target_std)))


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z = z + GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def raw_ints(seed: int, tensor_id: int, index: np.ndarray, mode: int = NORMAL) -> np.ndarray:
    """Integer draws v for the given flat element indices (int64 array)."""
    index = np.asarray(index, dtype=np.uint64)
    key = (np.uint64(seed & 0xFF) << np.uint64(56)) ^ (np.uint64(tensor_id & 0xFF) << np.uint64(48)) ^ index
    h = splitmix64(key)
    if mode == DYADIC:
        return (h % np.uint64(9)).astype(np.int64) - 4
    s = (h & np.uint64(0xFFFF)) + ((h >> np.uint64(16)) & np.uint64(0xFFFF)) \
        + ((h >> np.uint64(32)) & np.uint64(0xFFFF)) + (h >> np.uint64(48))
    return s.astype(np.int64) - 131070


def values_f32(seed, tensor_id, index, e, mode=NORMAL) -> np.ndarray:
    """v * 2**-e as float32 (exact: |v| < 2**18)."""
    v = raw_ints(seed, tensor_id, index, mode)
    return np.ldexp(v.astype(np.float32), -e).astype(np.float32)


def f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (finite inputs)."""
    b = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return b.astype(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    """Exact decode of bf16 bit patterns."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def gen_bf16_bits(seed, tensor_id, shape, e, mode=NORMAL, index=None) -> np.ndarray:
    n = int(np.prod(shape))
    idx = np.arange(n, dtype=np.int64) if index is None else np.asarray(index, dtype=np.int64)
    return f32_to_bf16_bits(values_f32(seed, tensor_id, idx, e, mode)).reshape(shape)


def gen_rows_bf16_bits(seed, tensor_id, rows, ncols, e, mode=NORMAL) -> np.ndarray:
    """Random access: only the requested rows of a [*, ncols] tensor."""
    rows = np.asarray(rows, dtype=np.int64)
    idx = (rows[:, None] * ncols + np.arange(ncols, dtype=np.int64)[None, :]).reshape(-1)
    return f32_to_bf16_bits(values_f32(seed, tensor_id, idx, e, mode)).reshape(len(rows), ncols)


def gen_rows_f32(seed, tensor_id, rows, ncols, e, mode=NORMAL) -> np.ndarray:
    rows = np.asarray(rows, dtype=np.int64)
    idx = (rows[:, None] * ncols + np.arange(ncols, dtype=np.int64)[None, :]).reshape(-1)
    return values_f32(seed, tensor_id, idx, e, mode).reshape(len(rows), ncols)


def default_exponents(d: int, d_ff: int, mode: int = NORMAL) -> dict:
    """Scale exponents per tensor (SURVEY.md 8(d) std table; P6 for dyadic)."""
    if mode == DYADIC:
        return {TID_X: 2, TID_SUBKEYS: 6, TID_W: 6, TID_V: 2, TID_W_GATE_UP: 6, TID_W_DOWN: 6}
    return {
        TID_X: scale_exponent(1.0),
        TID_SUBKEYS: scale_exponent(1.0 / math.sqrt(d)),
        TID_W: scale_exponent(1.0 / math.sqrt(d)),
        TID_V: scale_exponent(1.0),
        TID_W_GATE_UP: scale_exponent(1.0 / math.sqrt(d)),
        TID_W_DOWN: scale_exponent(1.0 / math.sqrt(max(d_ff, 1))),
    }


# ---------------------------------------------------------------- C host twin (speed only)
_HOST_SO = None


def build_host(force: bool = False) -> str:
    """Compile synth/synth_host.c (gcc, no CUDA) into synth/libsynth_host.so."""
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    src, so = os.path.join(here, "synth_host.c"), os.path.join(here, "libsynth_host.so")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", so, src, "-lm"])
    return so


def _host_lib():
    global _HOST_SO
    if _HOST_SO is None:
        import ctypes
        lib = ctypes.CDLL(build_host())
        P = ctypes.c_void_p
        lib.synth_rows_f64.argtypes = [ctypes.c_uint64, ctypes.c_uint64, P, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int]
        lib.synth_rows_f64.restype = None
        _HOST_SO = lib
    return _HOST_SO


def rows_f64(seed, tensor_id, rows, ncols, e, mode=NORMAL, bf16=True, nthreads=None) -> np.ndarray:
    """Decoded (exact float64) rows of a [*, ncols] tensor stored as bf16 (or fp32),
    computed by the C twin; identical to bf16_bits_to_f64(gen_rows_bf16_bits(...))
    (resp. gen_rows_f32(...).astype(float64))."""
    import os
    rows = np.ascontiguousarray(rows, dtype=np.int64).reshape(-1)
    out = np.empty((len(rows), ncols), dtype=np.float64)
    if len(rows) and ncols:
        _host_lib().synth_rows_f64(seed, tensor_id, rows.ctypes.data, len(rows), ncols, e, mode, int(bf16),
                                   out.ctypes.data, nthreads or os.cpu_count() or 1)
    return out
