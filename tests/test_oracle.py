"""Pins for the CPU oracle (-m "not gpu").  Each test pins an oracle function to
something other than itself: closed forms, exact integer / rational arithmetic,
brute force on tiny inputs, invariants, or SPEC worked examples
(tests/golden/spec_examples.json, each with its citation).
"Oracle pins" for which test pins which function."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _exact_topk(sr, sc, K):
    """Independent brute force with exact rational keys (Python Fractions)."""
    Nr, Nc = len(sr), len(sc)
    cells = [(Fraction(float(sr[i])) + Fraction(float(sc[j])), i * Nc + j)
             for i in range(Nr) for j in range(Nc)]
    cells.sort(key=lambda t: (-t[0], t[1]))
    return cells[:K + 1]


def _rand_logits(rng, T, Nr, Nc, kind):
    if kind == "cont":
        return rng.standard_normal((T, Nr + Nc)).astype(np.float32)
    if kind == "dyadic":  # heavy exact ties
        return (rng.integers(-3, 4, (T, Nr + Nc)) / 4.0).astype(np.float32)
    # rounding-adversarial: near-equal values differing in the last bits
    base = rng.integers(-2, 3, (T, Nr + Nc)).astype(np.float32)
    eps = rng.integers(-2, 3, (T, Nr + Nc)).astype(np.float32) * np.float32(2.0 ** -25)
    return (base + eps).astype(np.float32)


# ---- P1: brute force == exact rational brute force (tiny inputs) -----------------
@pytest.mark.parametrize("kind", ["cont", "dyadic", "adv"])
def test_bruteforce_matches_exact_rational(kind):
    rng = np.random.default_rng(7)
    for _ in range(60):
        Nr, Nc = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        K = int(rng.integers(1, Nr * Nc + 1))
        lg = _rand_logits(rng, 1, Nr, Nc, kind)
        r = oracle.route(lg, Nr, Nc, K, method=oracle.BRUTE, nthreads=1)
        ex = _exact_topk(lg[0, :Nr], lg[0, Nr:], K)
        assert list(r["idx"][0]) == [n for _, n in ex[:K]]
        if K < Nr * Nc:
            assert r["gap"][0] == pytest.approx(float(ex[K - 1][0] - ex[K][0]), abs=1e-12)


def test_exact_key_minimal_counterexample():
    """A.4: s_r=[0, 2^-25], s_c=[1], K=1.  fp32-rounded keys tie; exact keys do not."""
    lg = np.array([[0.0, 2.0 ** -25, 1.0]], dtype=np.float32)
    for m in (oracle.BRUTE, oracle.PRODUCT):
        assert oracle.route(lg, 2, 1, 1, method=m)["idx"][0, 0] == 1


# ---- P2: product == brute force == block-merge (>= 1000 instances) ---------------
@pytest.mark.parametrize("kind", ["cont", "dyadic", "adv"])
def test_product_equals_bruteforce(kind):
    rng = np.random.default_rng({"cont": 1, "dyadic": 2, "adv": 3}[kind])
    n = 0
    for _ in range(400):
        Nr, Nc = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        K = int(rng.integers(1, Nr * Nc + 1))
        lg = _rand_logits(rng, 3, Nr, Nc, kind)
        b = oracle.route(lg, Nr, Nc, K, method=oracle.BRUTE, nthreads=1)
        p = oracle.route(lg, Nr, Nc, K, method=oracle.PRODUCT, nthreads=1)
        m = oracle.route(lg, Nr, Nc, K, method=oracle.BLOCKMERGE, bsel=max(K + 1, 5), nthreads=1)
        for o in (p, m):
            np.testing.assert_array_equal(o["idx"], b["idx"])
            np.testing.assert_array_equal(o["gate"], b["gate"])
            np.testing.assert_array_equal(o["gap"], b["gap"])
        n += 3
    assert n >= 1000


def test_product_equals_bruteforce_larger():
    rng = np.random.default_rng(11)
    for Nr, Nc, K in [(64, 64, 1), (64, 64, 16), (32, 32, 8), (16, 48, 64), (256, 256, 16)]:
        lg = rng.standard_normal((4, Nr + Nc)).astype(np.float32)
        b = oracle.route(lg, Nr, Nc, K, method=oracle.BRUTE)
        p = oracle.route(lg, Nr, Nc, K, method=oracle.PRODUCT)
        np.testing.assert_array_equal(p["idx"], b["idx"])


# ---- P3: closed forms --------------------------------------------------------------
def test_k1_is_argmax_pair():
    rng = np.random.default_rng(5)
    lg = rng.standard_normal((20, 9 + 13)).astype(np.float32)
    r = oracle.route(lg, 9, 13, 1)
    for t in range(20):
        i, j = int(np.argmax(lg[t, :9])), int(np.argmax(lg[t, 9:]))
        assert r["idx"][t, 0] == i * 13 + j
        assert r["gate"][t, 0] == 1.0


def test_single_row_reduces_to_column_topk():
    rng = np.random.default_rng(6)
    lg = rng.standard_normal((10, 1 + 40)).astype(np.float32)
    r = oracle.route(lg, 1, 40, 7)
    for t in range(10):
        order = sorted(range(40), key=lambda j: (-lg[t, 1 + j], j))[:7]
        assert list(r["idx"][t]) == order


def test_zero_input_uniform():
    """x = 0 -> all keys 0 -> ids [0..K), gates 1/K (reading Q20)."""
    x = np.zeros((3, 16))
    sub = np.random.default_rng(0).standard_normal((1, 8 + 8, 16)).astype(np.float32)
    lg = oracle.logits(x, sub)
    r = oracle.route(lg.reshape(3, 16), 8, 8, 5)
    for t in range(3):
        assert list(r["idx"][t]) == [0, 1, 2, 3, 4]
        np.testing.assert_allclose(r["gate"][t], 0.2, rtol=0, atol=1e-15)


def test_uniform_tiebreak_golden():
    g = GOLD["uniform_tiebreak"]
    lg = np.zeros((1, g["n_rows"] + g["n_cols"]), np.float32)
    for m in (oracle.BRUTE, oracle.PRODUCT, oracle.BLOCKMERGE):
        assert list(oracle.route(lg, g["n_rows"], g["n_cols"], g["K"], method=m, bsel=4)["idx"][0]) == g["expected"]


def test_gates_two_golden():
    g = GOLD["gates_two"]
    lg = np.array([[g["scores"][0], g["scores"][1], 0.0]], dtype=np.float32)
    r = oracle.route(lg, 2, 1, 2)
    np.testing.assert_allclose(r["gate"][0], g["expected"], atol=1e-7)  # fp32 logits


def test_logsoftmax_golden_via_scores():
    g = GOLD["logsoftmax_two"]
    lg = np.array([[g["s"][0], g["s"][1], 0.0]], dtype=np.float32)
    r = oracle.route(lg, 2, 1, 2)
    # score = p_r[i] + p_c[j], p_c = log(1) = 0; sorted desc -> [ln 3/4, ln 1/4]
    np.testing.assert_allclose(r["score"][0], [g["expected"][1], g["expected"][0]], atol=1e-7)


def test_scores_are_log_probabilities_of_whole_halves_k_lt_n():
    """score = kappa - lse_r - lse_c with each lse over the WHOLE half (Eq.LSM,
    PAPER:215-219), not over the selected keys: rows with softmax probabilities
    [.1, .2, .3, .4], columns [.5, .5], K = 3 < N = 8.  Closed form: the top 3 cells
    are (3,0), (3,1) (exact tie: lower flat id 6 first, Q7), (2,0); scores are
    log(p_r p_c) = log .2, log .2, log .15; gates = softmax over the selected keys
    (Eq.Gate) = [4, 4, 3] / 11.  An lse over the selected keys only would give
    log(4/11) instead."""
    lg = np.array([[np.log(1.0), np.log(2.0), np.log(3.0), np.log(4.0), 0.0, 0.0]], dtype=np.float32)
    for m in (oracle.BRUTE, oracle.PRODUCT, oracle.BLOCKMERGE):
        r = oracle.route(lg, 4, 2, 3, method=m, bsel=3)
        assert list(r["idx"][0]) == [6, 7, 4]
        np.testing.assert_allclose(r["score"][0], np.log([0.2, 0.2, 0.15]), atol=1e-6)
        np.testing.assert_allclose(r["gate"][0], np.array([4, 4, 3]) / 11.0, atol=1e-6)
    # a second shape: 3 x 3 grid with K = 2, rows [.5, .25, .25], columns [.7, .2, .1]
    lg = np.array([[np.log(2.0), 0.0, 0.0, np.log(7.0), np.log(2.0), np.log(1.0)]], dtype=np.float32)
    r = oracle.route(lg, 3, 3, 2)
    assert list(r["idx"][0]) == [0, 3]  # (0,0) .35, then (1,0) and (2,0) tie at .175: id 3 < 6
    np.testing.assert_allclose(r["score"][0], np.log([0.35, 0.175]), atol=1e-6)
    assert r["gap"][0] == 0.0  # K-th and (K+1)-th keys are exactly equal


# ---- P4: invariants ----------------------------------------------------------------
def test_shift_invariance_and_normalisation():
    rng = np.random.default_rng(9)
    lg = (rng.integers(-64, 64, (50, 12 + 10)) / 16.0).astype(np.float32)
    r0 = oracle.route(lg, 12, 10, 6)
    lg2 = lg.copy()
    lg2[:, :12] += np.float32(0.75)  # dyadic shift: exact in fp32
    lg2[:, 12:] -= np.float32(2.5)
    r1 = oracle.route(lg2, 12, 10, 6)
    np.testing.assert_array_equal(r0["idx"], r1["idx"])
    np.testing.assert_allclose(r0["gate"], r1["gate"], atol=1e-12)
    np.testing.assert_allclose(r0["score"], r1["score"], atol=1e-12)  # log-probs absorb shift
    np.testing.assert_allclose(r0["gate"].sum(1), 1.0, atol=1e-12)
    for t in range(50):
        assert len(set(r0["idx"][t])) == 6
        assert np.all(np.diff(r0["score"][t]) <= 0)


# ---- O1 logits pinned by exact integer arithmetic (P6 + normal mode) ---------------
@pytest.mark.parametrize("mode", [synth.NORMAL, synth.DYADIC])
def test_logits_exact_integer(mode):
    d, L, h, R = 64, 5, 2, 24
    ex = synth.default_exponents(d, 0, mode)
    xb = synth.gen_bf16_bits(3, synth.TID_X, (L, d), ex[synth.TID_X], mode)
    sb = synth.gen_bf16_bits(3, synth.TID_SUBKEYS, (h, R, d), ex[synth.TID_SUBKEYS], mode)
    x, s = synth.bf16_bits_to_f64(xb), synth.bf16_bits_to_f64(sb)
    out = oracle.logits(x, s)
    # integers in units of 2^-e: exact int64 dot products, then one rounding to fp32
    xi = np.rint(np.ldexp(x, ex[synth.TID_X])).astype(np.int64)
    si = np.rint(np.ldexp(s, ex[synth.TID_SUBKEYS])).astype(np.int64)
    assert np.array_equal(np.ldexp(xi.astype(np.float64), -ex[synth.TID_X]), x)
    for l in range(L):
        for hh in range(h):
            for r in range(R):
                acc = int(np.dot(xi[l], si[hh, r]))  # exact (< 2^53)
                v = float(Fraction(acc, 2 ** (ex[synth.TID_X] + ex[synth.TID_SUBKEYS])))
                assert out[l, hh, r] == np.float32(v)


# ---- Q9: logits are RN32 of the exact dot product -----------------------------------
def _rn32_of_fraction(fr):
    """Round a rational to the nearest fp32 (ties to even) with Python integers only."""
    if fr == 0:
        return 0.0
    neg, a = fr < 0, abs(fr)
    e = a.numerator.bit_length() - a.denominator.bit_length() - 24
    while a / Fraction(2) ** e >= 2 ** 24:
        e += 1
    while a / Fraction(2) ** e < 2 ** 23:
        e -= 1
    q = a / Fraction(2) ** e
    n = q.numerator // q.denominator
    rem = q - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    v = float(np.float32(n * 2.0 ** e))
    assert Fraction(v) == n * Fraction(2) ** e  # representable: the rounding above was the only one
    return -v if neg else v


def _exact_dot(x, w):
    return sum((Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, w)), Fraction(0))


def test_exact_dot_random_vs_fractions():
    rng = np.random.default_rng(31)
    for trial in range(300):
        d = int(rng.integers(1, 80))
        if trial % 3 == 0:  # bf16 values of the generator's kind
            x = synth.bf16_bits_to_f64(synth.f32_to_bf16_bits(rng.standard_normal(d).astype(np.float32)))
            w = synth.bf16_bits_to_f64(synth.f32_to_bf16_bits((rng.standard_normal(d) / 8).astype(np.float32)))
        else:  # fp32 values spanning many binades
            x = (rng.standard_normal(d) * 2.0 ** rng.integers(-12, 12, d)).astype(np.float32).astype(np.float64)
            w = (rng.standard_normal(d) * 2.0 ** rng.integers(-12, 12, d)).astype(np.float32).astype(np.float64)
        assert oracle.exact_dot(x, w) == _rn32_of_fraction(_exact_dot(x, w))


def test_exact_dot_double_rounding_cases():
    """1 + 2^-24 + 2^-60: fp64 accumulation drops 2^-60 and then ties to even (1.0);
    the exact value lies above the fp32 midpoint, so RN32 gives 1 + 2^-23."""
    one = np.ones(3)
    assert oracle.exact_dot([1.0, 2.0 ** -24, 2.0 ** -60], one) == 1.0 + 2.0 ** -23
    assert oracle.exact_dot([1.0, 2.0 ** -24, -(2.0 ** -60)], one) == 1.0  # just below: down
    assert oracle.exact_dot([1.0, 2.0 ** -24], [1.0, 1.0]) == 1.0  # exact tie: to even
    assert oracle.exact_dot([1.0 + 2.0 ** -23, 2.0 ** -24], [1.0, 1.0]) == 1.0 + 2.0 ** -22  # tie: to even (up)
    assert oracle.exact_dot([3.0, -3.0], [5.0, 5.0]) == 0.0
    # a cancellation that fp64 sequential summation gets wrong
    x, w = [2.0 ** 40, 1.0, -(2.0 ** 40)], [1.0, 2.0 ** -30, 1.0]
    assert oracle.exact_dot(x, w) == 2.0 ** -30
    # contract: fp32-representable inputs only; anything else is reported as NaN
    assert np.isnan(oracle.exact_dot([0.1], [1.0]))
    assert np.isnan(oracle.exact_dot([2.0 ** 100, 2.0 ** -100], [1.0, 1.0]))


def test_logits_row_integer_path_vs_fractions():
    """oracle.logits writes each row once as integers at its finest exponent and sums
    the products in int64 / int128 (rows that do not fit fall back to the per-dot
    routine): every logit must still be RN32 of the exact Fraction dot product,
    for narrow rows (int64 sums), wide rows (int128 sums) and rows beyond 62-bit
    integers (fallback), and for the double-rounding and cancellation cases."""
    rng = np.random.default_rng(77)
    d = 40
    rows = []
    for kind in range(6):
        for _ in range(3):
            if kind == 0:  # bf16 generator-like
                v = synth.bf16_bits_to_f64(synth.f32_to_bf16_bits(rng.standard_normal(d).astype(np.float32)))
            elif kind == 1:  # fp32 over +-12 binades: int128 sums
                v = (rng.standard_normal(d) * 2.0 ** rng.integers(-12, 12, d)).astype(np.float32).astype(np.float64)
            elif kind == 2:  # exponent spread > 62 bits: fallback route
                v = (rng.standard_normal(d) * 2.0 ** rng.integers(-50, 50, d)).astype(np.float32).astype(np.float64)
            elif kind == 3:  # zeros and a zero row
                v = np.where(rng.random(d) < 0.5, 0.0, rng.integers(-4, 5, d) / 64.0)
            elif kind == 4:
                v = np.zeros(d)
            else:  # 1 + 2^-24 + 2^-60 padded: the double-rounding case inside a longer row
                v = np.zeros(d)
                v[:3] = [1.0, 2.0 ** -24, 2.0 ** -60]
            rows.append(v)
    X = np.array(rows)
    W = np.concatenate([X[::-1], np.ones((1, d))])[None]  # [1][R][d], includes the all-ones row
    got = oracle.logits(X, W)
    for i in range(X.shape[0]):
        for r in range(W.shape[1]):
            per_dot = oracle.exact_dot(X[i], W[0, r])
            if np.isnan(per_dot):  # beyond the 128-bit accumulator: NaN by contract, on both routes
                assert np.isnan(got[i, 0, r]), (i, r)
                continue
            want = _rn32_of_fraction(_exact_dot(X[i], W[0, r]))
            assert got[i, 0, r] == want == per_dot, (i, r, got[i, 0, r], want)


# ---- P5: schedule + executor identity ----------------------------------------------
def test_schedule_golden():
    g = GOLD["schedule_example"]
    ids = np.array(g["ids"], np.int32).reshape(-1)
    toks = np.repeat(np.arange(2), 2).astype(np.int32)
    p = oracle.schedule(ids, np.ones(4), toks, 0, 10)
    assert list(p["active"]) == g["active"]
    assert math.ceil(p["n_active"] / g["B"]) == g["n_groups"]
    assert list(p["sorted_token"]) == g["expected_sorted_token"]


def test_schedule_grouped_golden():
    g = GOLD["schedule_example_grouped"]
    ids = np.array(g["ids"], np.int32).reshape(-1)
    toks = np.repeat(np.arange(2), 2).astype(np.int32)
    p = oracle.schedule(ids, np.ones(4), toks, 0, 10, B=g["B"])
    assert list(p["sorted_token"]) == g["expected_sorted_token"]
    assert list(p["sorted_expert"]) == g["expected_sorted_expert"]
    assert list(p["run_offsets"]) == g["expected_run_offsets"]


@pytest.mark.parametrize("B,nblk", [(1, 1), (2, 1), (3, 1), (7, 1), (1000, 1), (3, 2), (7, 3)])
def test_schedule_grouped_properties(B, nblk):
    rng = np.random.default_rng(40 + B)
    L, HK, N = 60, 5, 41
    ids = rng.integers(0, N, (L, HK)).astype(np.int32)
    gates = rng.random((L, HK))
    toks = np.repeat(np.arange(L), HK).astype(np.int32)
    tpb = HK * -(-L // nblk) if nblk > 1 else 0
    for (b, e) in [(0, N), (7, 30)]:
        p = oracle.schedule(ids, gates, toks, b, e, B=B, tpb=tpb)
        fl = ids.reshape(-1)
        sel = (fl >= b) & (fl < e)
        active = sorted(set((fl[sel] - b).tolist()))
        assert list(p["active"]) == active
        grp = {ex: i // B for i, ex in enumerate(active)}
        # multiset conservation
        want = sorted(zip(toks[sel], fl[sel] - b, gates.reshape(-1)[sel]))
        got = sorted(zip(p["sorted_token"], p["sorted_expert"], p["sorted_gate"]))
        assert got == want
        # sorted by (token block, q, l) (Eq.Sort per token block)
        blk = (lambda l: l // (tpb // HK)) if tpb else (lambda l: 0)
        keys = [(blk(l), grp[ex], l) for ex, l in zip(p["sorted_expert"], p["sorted_token"])]
        assert keys == sorted(keys)
        assert len(set(grp.values())) == -(-len(active) // B)  # N_groups = ceil(|E_active| / B)
        # runs partition the plan into maximal constant (q, l) stretches
        ro = list(p["run_offsets"]) + [len(keys)]
        for r in range(len(ro) - 1):
            assert len(set(keys[ro[r]:ro[r + 1]])) == 1
            if r:
                assert keys[ro[r]] != keys[ro[r] - 1]
        if B == 1 and nblk == 1:  # expert-major: segment of e is [offsets[e], offsets[e+1])
            for ex in active:
                seg = p["sorted_expert"][p["offsets"][ex]:p["offsets"][ex + 1]]
                assert np.all(seg == ex)


@pytest.mark.parametrize("B,tpb", [(1, 0), (4, 0), (64, 0), (4, 9 * 7)])
def test_grouped_executor_equals_token_centric(B, tpb):
    rng = np.random.default_rng(50 + B)
    L, d, N, HK = 48, 24, 300, 9
    x = rng.standard_normal((L, d))
    W, V = rng.standard_normal((N, d)), rng.standard_normal((N, d))
    ids = np.stack([rng.choice(N, HK, replace=False) for _ in range(L)]).astype(np.int32)
    g = rng.random((L, HK))
    yt = oracle.routed_token_centric(x, W, V, ids, g)
    p = oracle.schedule(ids, g, np.repeat(np.arange(L), HK), 0, N, B=B, tpb=tpb)
    yg = oracle.routed_grouped(x, W, V, p)
    assert np.max(np.abs(yt - yg)) <= 1e-10 * max(1.0, np.max(np.abs(yt)))


def test_schedule_properties():
    rng = np.random.default_rng(4)
    L, HK, N = 40, 6, 37
    ids = rng.integers(0, N, (L, HK)).astype(np.int32)
    gates = rng.random((L, HK))
    toks = np.repeat(np.arange(L), HK).astype(np.int32)
    for (b, e) in [(0, N), (5, 20)]:
        p = oracle.schedule(ids, gates, toks, b, e)
        sel = (ids.reshape(-1) >= b) & (ids.reshape(-1) < e)
        # multiset conservation
        want = sorted(zip(toks[sel], ids.reshape(-1)[sel] - b, gates.reshape(-1)[sel]))
        got = []
        for ee in range(e - b):
            s, t = p["offsets"][ee], p["offsets"][ee + 1]
            assert np.all(np.diff(p["sorted_token"][s:t]) >= 0)  # tokens ascend
            got += [(p["sorted_token"][q], ee, p["sorted_gate"][q]) for q in range(s, t)]
        assert sorted(got) == want
        assert list(p["active"]) == [ee for ee in range(e - b) if p["offsets"][ee + 1] > p["offsets"][ee]]


@pytest.mark.parametrize("act", [0, 1])
def test_token_centric_equals_expert_centric(act):
    rng = np.random.default_rng(12)
    for L, d, N, HK in [(1, 8, 5, 1), (16, 32, 64, 8), (64, 16, 1024, 8), (30, 24, 7, 7)]:
        x = rng.standard_normal((L, d))
        W, V = rng.standard_normal((N, d)), rng.standard_normal((N, d))
        ids = np.stack([rng.choice(N, HK, replace=(HK > N)) for _ in range(L)]).astype(np.int32)
        g = rng.random((L, HK))
        yt = oracle.routed_token_centric(x, W, V, ids, g, act)
        p = oracle.schedule(ids, g, np.repeat(np.arange(L), HK), 0, N)
        ye = oracle.routed_expert_centric(x, W, V, p, act)
        assert np.max(np.abs(yt - ye)) <= 1e-10 * max(1.0, np.max(np.abs(yt)))


def test_atomic_expert_golden():
    g = GOLD["silu_atomic"]
    y = oracle.routed_token_centric(np.array([g["x"]]), np.array([g["w"]]), np.array([g["v"]]),
                                    np.array([[0]]), np.array([[1.0]]))
    np.testing.assert_allclose(y[0], g["expected"], rtol=0, atol=1e-15)


def test_orthogonal_input_zero():
    y = oracle.routed_token_centric(np.array([[1.0, 0.0]]), np.array([[0.0, 3.0]]),
                                    np.array([[5.0, 7.0]]), np.array([[0]]), np.array([[1.0]]))
    assert np.all(y == 0.0)


# ---- P8: linearity / convexity -----------------------------------------------------
def test_linearity_in_V_and_convexity():
    rng = np.random.default_rng(13)
    L, d, N, HK = 8, 16, 50, 5
    x = rng.standard_normal((L, d))
    W, V = rng.standard_normal((N, d)), rng.standard_normal((N, d))
    ids = np.stack([rng.choice(N, HK, replace=False) for _ in range(L)]).astype(np.int32)
    g = rng.random((L, HK)); g /= g.sum(1, keepdims=True)
    y1 = oracle.routed_token_centric(x, W, V, ids, g)
    for c in (0.0, 2.0, -1.0):
        assert np.max(np.abs(oracle.routed_token_centric(x, W, c * V, ids, g) - c * y1)) <= 1e-10
    # all atomic outputs equal u (identity act, z == 1) -> routed == u (gates sum to 1)
    x1 = np.zeros((L, d)); x1[:, 0] = 1.0
    W1 = np.zeros((N, d)); W1[:, 0] = 1.0
    u = rng.standard_normal(d)
    y = oracle.routed_token_centric(x1, W1, np.tile(u, (N, 1)), ids, g, act=1)
    np.testing.assert_allclose(y, np.tile(u, (L, 1)), atol=1e-12)


# ---- P9: shared MLP --------------------------------------------------------------
def test_shared_mlp_golden_and_zero():
    g = GOLD["shared_mlp_hand"]
    y = oracle.shared_mlp(np.array([g["x"]]), np.array(g["w_gu"]), np.array(g["w_down"]))
    np.testing.assert_allclose(y[0], g["expected"], rtol=1e-15)
    rng = np.random.default_rng(1)
    assert np.all(oracle.shared_mlp(np.zeros((2, 8)), rng.standard_normal((12, 8)),
                                    rng.standard_normal((8, 6))) == 0.0)


def test_shared_mlp_matches_numpy_composition():
    """Cross-check against the matrix form silu(xWg^T)*(xWu^T) Wd^T (numpy BLAS, fp64)."""
    rng = np.random.default_rng(2)
    x, wgu, wd = rng.standard_normal((7, 12)), rng.standard_normal((2 * 5, 12)), rng.standard_normal((12, 5))
    u, v = x @ wgu[:5].T, x @ wgu[5:].T
    ref = (u / (1 + np.exp(-u)) * v) @ wd.T
    np.testing.assert_allclose(oracle.shared_mlp(x, wgu, wd), ref, rtol=1e-12, atol=1e-12)


# ---- layer composition -------------------------------------------------------------
def test_layer_composition_equals_steps():
    rng = np.random.default_rng(21)
    L, d, Nr, Nc, K, h, dff = 12, 16, 6, 5, 4, 2, 8
    x = rng.standard_normal((L, d)).astype(np.float32).astype(np.float64)
    sub = rng.standard_normal((h, Nr + Nc, d)).astype(np.float32).astype(np.float64)
    W, V = rng.standard_normal((Nr * Nc, d)), rng.standard_normal((Nr * Nc, d))
    wgu, wd = rng.standard_normal((2 * dff, d)), rng.standard_normal((d, dff))
    out = oracle.layer(x, sub, W, V, Nr, Nc, K, wgu, wd)
    lg = oracle.logits(x, sub)
    r = oracle.route(lg.reshape(L * h, -1), Nr, Nc, K, method=oracle.BRUTE)
    np.testing.assert_array_equal(out["idx"].reshape(L * h, K), r["idx"])
    yr = oracle.routed_token_centric(x, W, V, r["idx"].reshape(L, h * K), r["gate"].reshape(L, h * K))
    ys = oracle.shared_mlp(x, wgu, wd)
    np.testing.assert_allclose(out["y"], yr + ys, rtol=1e-12, atol=1e-12)
    # compact tables through id_map give the same result
    used = np.unique(out["idx"])
    idm = np.stack([used, np.arange(len(used))], 1)
    out2 = oracle.layer(x, sub, W[used], V[used], Nr, Nc, K, wgu, wd, id_map=idm)
    np.testing.assert_array_equal(out2["y"], out["y"])


# ---- P12: absolute layer values at the paper's width, from closed forms -------------
def test_layer_closed_forms_paper_width():
    """Eq.MoE at d = 2048, K = 512 (C3a's width and top-k) on a 64 x 64 grid, with expert
    tables built so that the routed branch has a closed form whatever the routing: with every
    w_e = w and v_e = u, Eq.Assemble gives y_routed = sum_heads sum_k g_k silu(x.w) u =
    h silu(x.w) u (Eq.Gate: the gates of a head sum to 1); with v_e = (e mod d)-th unit vector
    scaled by (e + 1), y_routed[j] = sum over the selected e with e mod d = j of
    g_e silu(x.w_e) (e + 1).  The shared branch is switched off (w_down = 0) or
    checked against numpy's matrix form."""
    rng = np.random.default_rng(12)
    L, d, Nr, Nc, K, h, dff = 3, 2048, 64, 64, 512, 2, 64
    N = Nr * Nc
    x = rng.standard_normal((L, d)).astype(np.float32).astype(np.float64)
    sub = rng.standard_normal((h, Nr + Nc, d)).astype(np.float32).astype(np.float64) / 32
    w = rng.standard_normal(d) / 64
    u = rng.standard_normal(d)
    silu = lambda z: z / (1 + np.exp(-z))
    wgu = rng.standard_normal((2 * dff, d)) / 64
    out = oracle.layer(x, sub, np.tile(w, (N, 1)), np.tile(u, (N, 1)), Nr, Nc, K, wgu, np.zeros((d, dff)))
    np.testing.assert_allclose(out["y"], h * silu(x @ w)[:, None] * u[None, :], rtol=1e-10, atol=1e-12)
    # one-hot expert rows: the assembled output is the gate-weighted scatter of the selected ids
    W = rng.standard_normal((N, d)) / 64
    V = np.zeros((N, d))
    V[np.arange(N), np.arange(N) % d] = np.arange(N) + 1.0
    wd = rng.standard_normal((d, dff)) / 8
    out = oracle.layer(x, sub, W, V, Nr, Nc, K, wgu, wd)
    ref = np.zeros((L, d))
    for l in range(L):
        for head in range(h):
            for e, g in zip(out["idx"][l, head], out["gate"][l, head]):
                ref[l, e % d] += g * silu(x[l] @ W[e]) * (e + 1)
    hmid = silu(x @ wgu[:dff].T) * (x @ wgu[dff:].T)
    np.testing.assert_allclose(out["y"], ref + hmid @ wd.T, rtol=1e-9, atol=1e-9)
    assert np.allclose(out["gate"].sum(-1), 1.0) and len(set(out["idx"][0, 0])) == K


# ---- P11 generator sanity: |E_active| under near-uniform routing ---------------------
def test_active_expert_count_uniform_model():
    d, Nr, Nc, K, L = 64, 32, 32, 8, 256
    ex = synth.default_exponents(d, 0)
    x = synth.bf16_bits_to_f64(synth.gen_bf16_bits(0, synth.TID_X, (L, d), ex[synth.TID_X]))
    s = synth.bf16_bits_to_f64(synth.gen_bf16_bits(0, synth.TID_SUBKEYS, (1, Nr + Nc, d), ex[synth.TID_SUBKEYS]))
    r = oracle.route(oracle.logits(x, s).reshape(L, -1), Nr, Nc, K)
    n_act = len(np.unique(r["idx"]))
    N, M = Nr * Nc, L * K
    expect = N * (1 - (1 - 1 / N) ** M)
    assert abs(n_act - expect) / expect < 0.1  # within 0.1% at scale; loose at C1


def test_traffic_and_flop_formulas_golden():
    g = GOLD["traffic_counter"]
    assert 2 * g["d"] * g["L"] * g["K"] == g["expected"]
    f = GOLD["router_flops"]
    assert 2 * f["d"] * f["N"] == f["dense_flops"]
    rt = math.isqrt(f["N"])
    assert (2 * f["d"] * f["N"]) / (2 * f["d"] * (rt + rt)) == f["ratio"]


# ---------------------------------------------------------------- N1: load metrics and the dense-router ablation
def test_load_stats_closed_forms():
    """Expert Usage and Unevenness on cases with closed forms."""
    import math
    u, kl = oracle.load_stats(np.full(64, 3))          # uniform load: all used, KL = 0
    assert u == 1.0 and abs(kl) < 1e-15
    c = np.zeros(1000, np.int64)
    c[17] = 5                                          # one expert takes everything
    u, kl = oracle.load_stats(c)
    assert u == 1 / 1000 and abs(kl - math.log(1000)) < 1e-12
    u, kl = oracle.load_stats([2, 1, 1, 0])            # hand example: z = (1/2, 1/4, 1/4, 0)
    assert u == 0.75 and abs(kl - 0.5 * math.log(2)) < 1e-15
    assert oracle.load_stats(np.zeros(8, np.int64)) == (0.0, 0.0)


def test_load_stats_matches_textbook_kl():
    from scipy.stats import entropy
    rng = np.random.default_rng(3)
    c = rng.poisson(2.0, 5000)
    u, kl = oracle.load_stats(c)
    z = c / c.sum()
    assert u == np.count_nonzero(c) / c.size
    assert abs(kl - entropy(z, np.full(c.size, 1 / c.size))) < 1e-12


def test_dense_route_pins():
    """The 'w/o CPR' router: exact top-K by (value desc, id asc)."""
    rng = np.random.default_rng(5)
    s = rng.standard_normal((50, 300)).astype(np.float32)
    s[:, 100] = s[:, 7]                                 # exact ties: the lower id first
    s[3, :] = 0.25                                      # a row of equal values -> ids [0..K)
    r = oracle.dense_route(s, 12)
    for t in range(50):                                 # independent formulation: lexsort on (-value, id)
        order = np.lexsort((np.arange(300), -s[t].astype(np.float64)))[:12]
        np.testing.assert_array_equal(r["idx"][t], order)
    np.testing.assert_array_equal(r["idx"][3], np.arange(12))
    np.testing.assert_allclose(r["gate"].sum(1), 1.0, atol=1e-12)
    k1 = oracle.dense_route(s, 1)
    np.testing.assert_array_equal(k1["idx"][:, 0], np.argmax(s, 1))  # K = 1: the (first) arg-max
    g = oracle.dense_route(np.log(np.array([[0.6, 0.3, 0.1]], np.float32)), 2)["gate"][0]
    np.testing.assert_allclose(g, [0.6 / 0.9, 0.3 / 0.9], rtol=1e-6)  # softmax over the selected only
    sh = oracle.dense_route(s + np.float32(4.0), 12)   # shift invariance (exact in fp32 here)
    np.testing.assert_array_equal(sh["idx"][:3], r["idx"][:3])


# ---------------------------------------------------------------- N2: backward of the routed branch
@pytest.mark.parametrize("act", [0, 1])
def test_routed_bwd_matches_finite_differences(act):
    """Every gradient of oracle.routed_bwd against central differences of the
    forward oracle (loss = sum dy * y_routed), all in fp64."""
    rng = np.random.default_rng(11 + act)
    L, d, rows, HK = 5, 6, 9, 3
    x = rng.standard_normal((L, d))
    W = rng.standard_normal((rows, d)) * 0.5
    V = rng.standard_normal((rows, d))
    ids = np.stack([rng.choice(rows, HK, replace=False) for _ in range(L)]).astype(np.int32)
    ids[2] = ids[0]                                   # two tokens sharing experts
    g = rng.random((L, HK))
    dy = rng.standard_normal((L, d))
    grad = oracle.routed_bwd(x, W, V, ids, g, dy, act)

    def loss(x_, W_, V_, g_):
        return float((dy * oracle.routed_token_centric(x_, W_, V_, ids, g_, act)).sum())

    h = 1e-6
    for name, arr in (("dx", x), ("dW", W), ("dV", V), ("dgate", g)):
        fd = np.zeros_like(arr)
        for i in np.ndindex(arr.shape):
            p_, m_ = arr.copy(), arr.copy()
            p_[i] += h
            m_[i] -= h
            args_p = {"dx": (p_, W, V, g), "dW": (x, p_, V, g), "dV": (x, W, p_, g), "dgate": (x, W, V, p_)}[name]
            args_m = {"dx": (m_, W, V, g), "dW": (x, m_, V, g), "dV": (x, W, m_, g), "dgate": (x, W, V, m_)}[name]
            fd[i] = (loss(*args_p) - loss(*args_m)) / (2 * h)
        np.testing.assert_allclose(grad[name], fd, rtol=1e-6, atol=1e-7, err_msg=name)


def test_routed_bwd_closed_form():
    """d = 2, one task: x = [1, 0], w = [2, 0], v = [1, 1], g = 1, dy = [1, 0]:
    y = SiLU(2) v; dgate = SiLU(2) (dy . v) = SiLU(2); dV = SiLU(2) dy."""
    s2 = 2 / (1 + np.exp(-2.0))
    r = oracle.routed_bwd(np.array([[1.0, 0]]), np.array([[2.0, 0]]), np.array([[1.0, 1]]), np.array([[0]]),
                          np.array([[1.0]]), np.array([[1.0, 0]]))
    np.testing.assert_allclose(r["dgate"], [[s2]], rtol=1e-15)
    np.testing.assert_allclose(r["dV"], [[s2, 0]], rtol=1e-15)
    lg = 1 / (1 + np.exp(-2.0))
    sp = lg * (1 + 2 * (1 - lg))
    np.testing.assert_allclose(r["dx"], [[2 * sp, 0]], rtol=1e-14)   # dz = q sigma'(2) = sigma'(2); dx = dz w
    np.testing.assert_allclose(r["dW"], [[sp, 0]], rtol=1e-14)       # dW = dz x


def _fd(f, arr, h=1e-6):
    g = np.zeros_like(arr)
    for i in np.ndindex(arr.shape):
        p_, m_ = arr.copy(), arr.copy()
        p_[i] += h
        m_[i] -= h
        g[i] = (f(p_) - f(m_)) / (2 * h)
    return g


def test_router_bwd_matches_finite_differences():
    """loss = sum dgate * gate(x, sub) with the selected cells fixed (softmax over the
    selected keys, key = s_r + s_c, s = x . sub), against the analytic chain."""
    rng = np.random.default_rng(2)
    L, d, h, Nr, Nc, K = 3, 5, 2, 4, 3, 4
    x = rng.standard_normal((L, d))
    sub = rng.standard_normal((h, Nr + Nc, d))
    idx = np.stack([np.stack([rng.choice(Nr * Nc, K, replace=False) for _ in range(h)]) for _ in range(L)])
    idx = idx.astype(np.int32)
    dg = rng.standard_normal((L, h, K))

    def gates(x_, sub_):
        s = np.einsum("ld,hrd->lhr", x_, sub_)
        key = s[..., :Nr][np.arange(L)[:, None, None], np.arange(h)[None, :, None], idx // Nc] + \
            s[..., Nr:][np.arange(L)[:, None, None], np.arange(h)[None, :, None], idx % Nc]
        e = np.exp(key - key.max(-1, keepdims=True))
        return e / e.sum(-1, keepdims=True)

    g0 = gates(x, sub)
    dx, dsub = oracle.router_bwd(x, sub, Nr, Nc, idx, g0, dg)
    np.testing.assert_allclose(dx, _fd(lambda a: float((dg * gates(a, sub)).sum()), x), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(dsub, _fd(lambda a: float((dg * gates(x, a)).sum()), sub), rtol=1e-6, atol=1e-8)


def test_mlp_bwd_matches_finite_differences():
    rng = np.random.default_rng(4)
    L, d, dff = 3, 5, 4
    x = rng.standard_normal((L, d))
    wgu = rng.standard_normal((2 * dff, d)) * 0.5
    wdn = rng.standard_normal((d, dff)) * 0.5
    dy = rng.standard_normal((L, d))
    dx, dgu, ddn = oracle.mlp_bwd(x, wgu, wdn, dy)
    loss = lambda x_, a_, b_: float((dy * oracle.shared_mlp(x_, a_, b_)).sum())
    np.testing.assert_allclose(dx, _fd(lambda a: loss(a, wgu, wdn), x), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(dgu, _fd(lambda a: loss(x, a, wdn), wgu), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(ddn, _fd(lambda a: loss(x, wgu, a), wdn), rtol=1e-6, atol=1e-8)
