"""The seeded input generator's twins agree bit for bit (CPU).  The device twin
is checked against numpy in tests/test_gpu_parity.py::test_synth_device_matches_host."""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("mode", [synth.NORMAL, synth.DYADIC])
@pytest.mark.parametrize("bf16", [True, False])
@pytest.mark.parametrize("tid,e", [(synth.TID_X, 15), (synth.TID_W, 21), (synth.TID_V, 2)])
def test_c_twin_matches_numpy(mode, bf16, tid, e):
    rng = np.random.default_rng(tid * 7 + e)
    rows = np.concatenate([rng.integers(0, 1 << 22, 300), [0, 1, (1 << 22) - 1]])
    ncols = 2048 if tid != synth.TID_V else 72
    got = synth.rows_f64(3, tid, rows, ncols, e, mode, bf16=bf16, nthreads=4)
    if bf16:
        want = synth.bf16_bits_to_f64(synth.gen_rows_bf16_bits(3, tid, rows, ncols, e, mode))
    else:
        want = synth.gen_rows_f32(3, tid, rows, ncols, e, mode).astype(np.float64)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_c_twin_empty():
    assert synth.rows_f64(0, synth.TID_X, np.zeros(0, np.int64), 64, 15).shape == (0, 64)


def test_routing_counts_matches_loop():
    """The vectorised whole-batch counter agrees with the per-token-head loop of
    compare_routing (reading Q10) on equal, permuted, tied and wrong sets."""
    from tests.helpers import compare_routing, routing_counts
    rng = np.random.default_rng(0)
    T, nr, nc, K = 40, 6, 5, 4
    rows = rng.integers(-8, 8, (T, nr + nc)).astype(np.float32)
    key = rows[:, :nr, None].astype(np.float64) + rows[:, None, nr:]
    flat = key.reshape(T, -1)
    idx = np.argsort(-flat, -1, kind="stable")[:, :K].astype(np.int32)
    kk = np.take_along_axis(flat, idx, -1)
    g = np.exp(kk - kk.max(-1, keepdims=True))
    g /= g.sum(-1, keepdims=True)
    orc = dict(idx=idx, gate=g, key_hi=kk, key_lo=np.zeros_like(kk))
    gi, gg = idx.copy(), g.copy()
    gi[1] = gi[1][::-1]; gg[1] = gg[1][::-1]          # same set, other order
    nxt = np.argsort(-flat, -1, kind="stable")[:, K]
    gi[2, -1] = nxt[2]                                  # swapped in the (K+1)-th cell
    gi[3, 0] = nxt[3]                                   # swapped out the best cell
    a = compare_routing(gi, gg, orc, rows, nr, nc)
    b = routing_counts(gi, gg, orc, rows, nr, nc)
    assert {k: a[k] for k in ("mismatch", "allowed", "disallowed")} == \
           {k: b[k] for k in ("mismatch", "allowed", "disallowed")}
    assert b["mismatch"] == 2 and abs(a["gate_err"] - b["gate_err"]) < 1e-15
