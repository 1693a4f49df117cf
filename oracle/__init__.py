"""ctypes wrapper around oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package.  The product path
(paper_2602_05711_b200) never imports it; tests/test_abi_cpu.py::test_product_never_imports_oracle
enforces that.
See oracle/oracle.cpp for the citations of each function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

i64, i32, c_int = ctypes.c_int64, ctypes.c_int32, ctypes.c_int
P = ctypes.c_void_p


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
                               "-o", _SO, src])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        _lib.oracle_logits.argtypes = [i64, i64, i64, i64, P, P, P, c_int]
        _lib.oracle_exact_dot.argtypes = [P, P, i64]
        _lib.oracle_exact_dot.restype = ctypes.c_float
        _lib.oracle_route.argtypes = [i64, i64, i64, i64, P, c_int, i64, c_int, P, P, P, P, P, P]
        _lib.oracle_schedule.argtypes = [i64, P, P, P, i64, i64, i64, i64, P, P, P, P, P, P, P, P]
        _lib.oracle_routed_grouped.argtypes = [i64, i64, i64, i64, P, P, P, P, P, P, P, c_int, P]
        _lib.oracle_routed_token_centric.argtypes = [i64, i64, i64, P, P, P, P, P, c_int, P, c_int]
        _lib.oracle_routed_expert_centric.argtypes = [i64, i64, i64, P, P, P, P, P, P, c_int, P]
        _lib.oracle_shared_mlp.argtypes = [i64, i64, i64, P, P, P, P, c_int]
        _lib.oracle_load_stats.argtypes = [i64, P, P]
        _lib.oracle_dense_route.argtypes = [i64, i64, i64, P, c_int, P, P, P, P]
        _lib.oracle_routed_bwd.argtypes = [i64, i64, i64, P, P, P, P, P, P, c_int, i64, P, P, P, P]
        _lib.oracle_router_bwd.argtypes = [i64, i64, i64, i64, i64, i64, P, P, P, P, P, P, P]
        _lib.oracle_mlp_bwd.argtypes = [i64, i64, i64, P, P, P, P, P, P, P]
        _lib.oracle_layer.argtypes = [i64, i64, i64, i64, i64, i64, i64, P, P, P, P, P, i64, P, P,
                                      c_int, P, P, P, c_int]
        for f in ("oracle_logits", "oracle_route", "oracle_schedule", "oracle_routed_grouped",
                  "oracle_routed_token_centric",
                  "oracle_routed_expert_centric", "oracle_shared_mlp", "oracle_layer", "oracle_load_stats",
                  "oracle_dense_route", "oracle_routed_bwd", "oracle_router_bwd", "oracle_mlp_bwd"):
            getattr(_lib, f).restype = None
    return _lib


def _p(a):
    return a.ctypes.data_as(P) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def default_threads() -> int:
    return os.cpu_count() or 1


def exact_dot(x, w) -> float:
    """RN32 of the exact real dot product of two fp32-representable vectors (Q9)."""
    x, w = _f64(x).reshape(-1), _f64(w).reshape(-1)
    assert x.size == w.size
    return float(lib().oracle_exact_dot(_p(x), _p(w), x.size))


def logits(x, subkeys, nthreads=None):
    """x: [L][d], subkeys: [h][R][d] (exactly-decoded values) -> fp32 [L][h][R],
    each the RN32 of the exact dot product (reading Q9)."""
    x, subkeys = _f64(x), _f64(subkeys)
    L, d = x.shape
    h, R, _ = subkeys.shape
    out = np.empty((L, h, R), dtype=np.float32)
    lib().oracle_logits(L, d, h, R, _p(x), _p(subkeys), _p(out), nthreads or default_threads())
    return out


BRUTE, PRODUCT, BLOCKMERGE = 0, 1, 2


def route(logit_rows, n_rows, n_cols, K, method=PRODUCT, bsel=4096, nthreads=None):
    """logit_rows: [T][n_rows+n_cols] fp32 -> dict(idx, gate, score, key_hi, key_lo, gap)."""
    lg = np.ascontiguousarray(logit_rows, dtype=np.float32).reshape(-1, n_rows + n_cols)
    T = lg.shape[0]
    out = dict(idx=np.empty((T, K), np.int32), gate=np.empty((T, K)), score=np.empty((T, K)),
               key_hi=np.empty((T, K)), key_lo=np.empty((T, K)), gap=np.empty(T))
    lib().oracle_route(T, n_rows, n_cols, K, _p(lg), method, bsel, nthreads or default_threads(),
                       _p(out["idx"]), _p(out["gate"]), _p(out["score"]), _p(out["key_hi"]),
                       _p(out["key_lo"]), _p(out["gap"]))
    return out


def routed_bwd(x, W, V, ids, gates, dy, act=0):
    """N2: gradients of the routed branch for fixed routing -> dict(dx, dW, dV, dgate)
    (dW, dV shaped like W, V; ids index their rows)."""
    x, W, V, gates, dy = _f64(x), _f64(W), _f64(V), _f64(gates), _f64(dy)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    L, d = x.shape
    HK = ids.size // max(L, 1)
    rows = W.shape[0]
    out = dict(dx=np.empty((L, d)), dW=np.empty((rows, d)), dV=np.empty((rows, d)), dgate=np.empty((L, HK)))
    lib().oracle_routed_bwd(L, d, HK, _p(x), _p(W), _p(V), _p(ids), _p(gates), _p(dy), act, rows, _p(out["dx"]),
                            _p(out["dW"]), _p(out["dV"]), _p(out["dgate"]))
    return out


def router_bwd(x, subkeys, n_rows, n_cols, idx, gate, dgate):
    """N2 router part: (dx [L][d], dsub [h][R][d]) for fixed selections idx [L][h][K]."""
    x, sub = _f64(x), _f64(subkeys)
    L, d = x.shape
    h = sub.shape[0]
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    K = idx.shape[-1]
    dx = np.zeros((L, d))
    dsub = np.empty(sub.shape)
    lib().oracle_router_bwd(L, d, h, n_rows, n_cols, K, _p(x), _p(sub), _p(idx), _p(_f64(gate)), _p(_f64(dgate)),
                            _p(dx), _p(dsub))
    return dx, dsub


def mlp_bwd(x, w_gu, w_down, dy):
    """N2 shared-MLP part: (dx, dw_gate_up, dw_down)."""
    x, w_gu, w_down, dy = _f64(x), _f64(w_gu), _f64(w_down), _f64(dy)
    L, d = x.shape
    dff = w_down.shape[1]
    dx = np.zeros((L, d))
    dgu = np.empty(w_gu.shape)
    ddn = np.empty(w_down.shape)
    lib().oracle_mlp_bwd(L, d, dff, _p(x), _p(w_gu), _p(w_down), _p(dy), _p(dx), _p(dgu), _p(ddn))
    return dx, dgu, ddn


def load_stats(counts):
    """(Expert Usage, Unevenness) of per-expert task counts."""
    c = np.ascontiguousarray(counts, dtype=np.int64).reshape(-1)
    out = np.zeros(2)
    lib().oracle_load_stats(c.size, _p(c), _p(out))
    return float(out[0]), float(out[1])


def dense_route(logit_rows, K, nthreads=None):
    """Ablation 'w/o CPR': exact top-K of dense scores [T][N] by (value
    desc, id asc); dict(idx, gate, key, gap)."""
    lg = np.ascontiguousarray(logit_rows, dtype=np.float32)
    T, N = lg.shape
    out = dict(idx=np.empty((T, K), np.int32), gate=np.empty((T, K)), key=np.empty((T, K)), gap=np.empty(T))
    lib().oracle_dense_route(T, N, K, _p(lg), nthreads or default_threads(), _p(out["idx"]), _p(out["gate"]),
                             _p(out["key"]), _p(out["gap"]))
    return out


def schedule(ids, gates, tokens, n_begin, n_end, B=1, tpb=0):
    """Expert-centric plan with group size B, scheduled in blocks
    of tpb consecutive tasks when tpb > 0; see oracle_schedule."""
    ids = np.ascontiguousarray(ids, dtype=np.int32).reshape(-1)
    gates = _f64(gates).reshape(-1)
    tokens = np.ascontiguousarray(tokens, dtype=np.int32).reshape(-1)
    M, n_loc = ids.size, n_end - n_begin
    offsets = np.empty(n_loc + 1, np.int32)
    st = np.empty(max(M, 1), np.int32)
    sg = np.empty(max(M, 1), np.float64)
    se = np.empty(max(M, 1), np.int32)
    ro = np.empty(max(M, 1), np.int32)
    active = np.empty(max(n_loc, 1), np.int32)
    na = np.zeros(1, np.int64)
    nr = np.zeros(1, np.int64)
    lib().oracle_schedule(M, _p(ids), _p(gates), _p(tokens), n_begin, n_end, B, tpb, _p(offsets), _p(st),
                          _p(sg), _p(se), _p(active), _p(na), _p(ro), _p(nr))
    m_loc = int(offsets[-1])
    return dict(offsets=offsets, sorted_token=st[:m_loc], sorted_gate=sg[:m_loc], sorted_expert=se[:m_loc],
                active=active[:int(na[0])], n_active=int(na[0]), run_offsets=ro[:int(nr[0])],
                n_runs=int(nr[0]), B=B)


def routed_grouped(x, W_loc, V_loc, plan, act=0):
    """Eq.Grouped run by run over a plan from schedule(...)."""
    x, W_loc, V_loc = _f64(x), _f64(W_loc), _f64(V_loc)
    L, d = x.shape
    ro = np.ascontiguousarray(plan["run_offsets"], dtype=np.int32)
    st = np.ascontiguousarray(plan["sorted_token"], dtype=np.int32)
    se = np.ascontiguousarray(plan["sorted_expert"], dtype=np.int32)
    sg = _f64(plan["sorted_gate"])
    y = np.empty((L, d))
    lib().oracle_routed_grouped(L, d, st.size, ro.size, _p(ro), _p(st), _p(se), _p(sg), _p(x), _p(W_loc),
                                _p(V_loc), act, _p(y))
    return y


def routed_token_centric(x, W, V, ids, gates, act=0, nthreads=None):
    """ids/gates: [L][HK] (ids index rows of W/V)."""
    x, W, V, gates = _f64(x), _f64(W), _f64(V), _f64(gates)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    L, d = x.shape
    HK = ids.shape[1] if ids.ndim == 2 else ids.size // max(L, 1)
    y = np.empty((L, d))
    lib().oracle_routed_token_centric(L, d, HK, _p(x), _p(W), _p(V), _p(ids), _p(gates), act,
                                      _p(y), nthreads or default_threads())
    return y


def routed_expert_centric(x, W_loc, V_loc, plan, act=0):
    x, W_loc, V_loc = _f64(x), _f64(W_loc), _f64(V_loc)
    L, d = x.shape
    off = np.ascontiguousarray(plan["offsets"], dtype=np.int32)
    st = np.ascontiguousarray(plan["sorted_token"], dtype=np.int32)
    sg = _f64(plan["sorted_gate"])
    y = np.empty((L, d))
    lib().oracle_routed_expert_centric(L, d, off.size - 1, _p(off), _p(st), _p(sg), _p(x),
                                       _p(W_loc), _p(V_loc), act, _p(y))
    return y


def shared_mlp(x, w_gu, w_down, nthreads=None):
    x, w_gu, w_down = _f64(x), _f64(w_gu), _f64(w_down)
    L, d = x.shape
    d_ff = w_down.shape[1]
    y = np.empty((L, d))
    lib().oracle_shared_mlp(L, d, d_ff, _p(x), _p(w_gu), _p(w_down), _p(y),
                            nthreads or default_threads())
    return y


def layer(x, subkeys, W, V, n_rows, n_cols, K, w_gu=None, w_down=None, act=0, id_map=None,
          nthreads=None):
    """Full layer forward (Eq.MoE).  subkeys: [h][n_rows+n_cols][d].
    id_map: optional int64 [n_map][2] sorted (flat id, row of W/V) for compact tables."""
    x, subkeys, W, V = _f64(x), _f64(subkeys), _f64(W), _f64(V)
    L, d = x.shape
    h = subkeys.shape[0]
    d_ff = 0 if w_down is None else w_down.shape[1]
    w_gu = _f64(w_gu) if d_ff else None
    w_down = _f64(w_down) if d_ff else None
    idm = None if id_map is None else np.ascontiguousarray(id_map, dtype=np.int64)
    y = np.empty((L, d))
    idx = np.empty((L, h, K), np.int32)
    gate = np.empty((L, h, K))
    lib().oracle_layer(L, d, n_rows, n_cols, K, h, d_ff, _p(x), _p(subkeys), _p(W), _p(V),
                       _p(idm), 0 if idm is None else idm.shape[0], _p(w_gu), _p(w_down), act,
                       _p(y), _p(idx), _p(gate), nthreads or default_threads())
    return dict(y=y, idx=idx, gate=gate)
