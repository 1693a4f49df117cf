"""Test harness helpers: host (numpy) regeneration of the seeded inputs and the
parity metrics of DESIGN.md ("Comparison protocol").  Holds no arithmetic of
the method: oracle values come from oracle/, GPU values from the library."""
from __future__ import annotations

import numpy as np

import synth


def host_rows(dims, seed, name, rows=None, mode=synth.NORMAL):
    """Exact float64 values of rows of an input tensor (regenerated on the host)."""
    ex = synth.default_exponents(dims.d, dims.d_ff, mode)
    R = dims.n_rows * dims.n_cols if getattr(dims, "router", 0) == 2 else dims.n_rows + dims.n_cols
    tid, ncols, nrows = {
        "x": (synth.TID_X, dims.d, None),
        "subkeys": (synth.TID_SUBKEYS, dims.d, dims.n_heads * R),
        "W": (synth.TID_W, dims.d, dims.n_rows * dims.n_cols),
        "V": (synth.TID_V, dims.d, dims.n_rows * dims.n_cols),
        "w_gate_up": (synth.TID_W_GATE_UP, dims.d, 2 * dims.d_ff),
        "w_down": (synth.TID_W_DOWN, dims.d_ff, dims.d),
    }[name]
    if rows is None:
        rows = np.arange(nrows)
    # the C twin of the generator (bit-identical to the numpy one: tests/test_synth.py::test_c_twin_matches_numpy)
    return synth.rows_f64(seed, tid, rows, ncols, ex[tid], mode, bf16=dims.dtype == 0)


def oracle_keys(logit_rows, n_rows, n_cols, ids):
    """Exact key (fp64 sum of the two fp32 logits; exact within the tolerance
    used for allowances) of flat ids for every token-head."""
    lg = logit_rows.astype(np.float64)
    i, j = ids // n_cols, ids % n_cols
    T = lg.shape[0]
    return lg[np.arange(T)[:, None], i] + lg[np.arange(T)[:, None], n_rows + j]


def compare_routing(gpu_idx, gpu_gate, orc, logit_rows, n_rows, n_cols, allow_gap=1e-6):
    """Set comparison per token-head (reading Q10).  Returns counts and the max
    gate error over token-heads whose sets match."""
    gi = np.asarray(gpu_idx).reshape(orc["idx"].shape)
    gg = np.asarray(gpu_gate).reshape(orc["idx"].shape)
    T, K = gi.shape
    mism = allowed = disallowed = 0
    gate_err = 0.0
    kappa_K = orc["key_hi"][:, K - 1] + orc["key_lo"][:, K - 1]
    for t in range(T):
        a, b = set(gi[t].tolist()), set(orc["idx"][t].tolist())
        if a == b:
            oi = {n: g for n, g in zip(orc["idx"][t], orc["gate"][t])}
            gate_err = max(gate_err, max(abs(oi[n] - g) for n, g in zip(gi[t], gg[t])))
            continue
        mism += 1
        diff = np.array(sorted(a ^ b), dtype=np.int64)
        kd = oracle_keys(logit_rows[t:t + 1], n_rows, n_cols, diff[None, :])[0]
        if np.all(np.abs(kd - kappa_K[t]) < allow_gap):
            allowed += 1
        else:
            disallowed += 1
    return dict(mismatch=mism, allowed=allowed, disallowed=disallowed, gate_err=gate_err)


def routing_counts(gpu_idx, gpu_gate, orc, logit_rows, n_rows, n_cols, allow_gap=1e-6):
    """compare_routing for whole batches: set equality is checked vectorised, the
    Q10 allowance only on the token-heads whose sets differ; the gate error is
    taken over all token-heads with equal sets."""
    gi = np.asarray(gpu_idx).reshape(orc["idx"].shape)
    gg = np.asarray(gpu_gate).reshape(orc["idx"].shape)
    og = np.argsort(gi, -1, kind="stable")
    oo = np.argsort(orc["idx"], -1, kind="stable")
    gs, os_ = np.take_along_axis(gi, og, -1), np.take_along_axis(orc["idx"], oo, -1)
    same = np.all(gs == os_, -1)
    gate_err = 0.0
    if same.any():
        d = np.abs(np.take_along_axis(gg, og, -1) - np.take_along_axis(orc["gate"], oo, -1))[same]
        gate_err = float(d.max())
    bad = np.flatnonzero(~same)
    r = dict(mismatch=0, allowed=0, disallowed=0, gate_err=gate_err, token_heads=int(gi.shape[0]))
    if len(bad):
        sub = {k: orc[k][bad] for k in ("idx", "gate", "key_hi", "key_lo")}
        c = compare_routing(gi[bad], gg[bad], sub, logit_rows[bad], n_rows, n_cols, allow_gap)
        r.update(mismatch=c["mismatch"], allowed=c["allowed"], disallowed=c["disallowed"])
    return r


def rel_errors(y, ref):
    """e_tok = max_l ||y_l - ref_l||_2 / ||ref_l||_2 ;  e_elt = max |d| / max(|ref|, rms(ref_l))
    (reading Q17)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = y - ref
    nr = np.linalg.norm(ref, axis=1)
    e_tok = float(np.max(np.linalg.norm(d, axis=1) / np.maximum(nr, 1e-30)))
    rms = nr / np.sqrt(ref.shape[1])
    e_elt = float(np.max(np.abs(d) / np.maximum(np.abs(ref), np.maximum(rms[:, None], 1e-30))))
    return e_tok, e_elt
