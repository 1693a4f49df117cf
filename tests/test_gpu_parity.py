"""GPU-vs-oracle parity through the C ABI (-m gpu).  Inputs are seeded and
synthetic (synth/); expected values come only from oracle/."""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth.cuda import make
from synth.workloads import make_inputs
from paper_2602_05711_b200 import configs, omnimoe as om
from tests.helpers import compare_routing, host_rows, rel_errors

pytestmark = pytest.mark.gpu


def _dims(name, **over):
    return configs.get(name, **over)


# ---------------------------------------------------------------- generator
@pytest.mark.parametrize("mode", [synth.NORMAL, synth.DYADIC])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_synth_device_matches_host(mode, dt):
    n = 100_003
    t = make((n,), dt, 5, synth.TID_W, 13, mode)
    idx = np.arange(n)
    if dt == torch.bfloat16:
        want = synth.gen_bf16_bits(5, synth.TID_W, (n,), 13, mode)
        got = t.view(torch.int16).cpu().numpy().view(np.uint16)
    else:
        want = synth.values_f32(5, synth.TID_W, idx, 13, mode).view(np.uint32)
        got = t.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- tcgen05 GEMM engine
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 520, 136), (1000, 2048, 1024), (77, 40, 8),
                                   (4096, 640, 1024)])
def test_gemm_tcgen05(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    C = om.gemm_bf16(A, B)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().T
    err = (C.double() - ref).abs().max().item()
    assert err <= 1e-5 * K ** 0.5 * ref.abs().max().item() + 1e-6, err


# ---------------------------------------------------------------- router
def _oracle_route(dims, seed, tokens, mode=synth.NORMAL, method=oracle.BRUTE):
    x = host_rows(dims, seed, "x", tokens, mode)
    sub = host_rows(dims, seed, "subkeys", None, mode).reshape(dims.n_heads, dims.n_rows + dims.n_cols, dims.d)
    lg = oracle.logits(x, sub)  # [T][h][R]
    rows = lg.reshape(-1, dims.n_rows + dims.n_cols)
    return oracle.route(rows, dims.n_rows, dims.n_cols, dims.top_k, method=method), rows


ROUTERS = [om.ROUTER_EXACT, om.ROUTER_EXACT_F64]


@pytest.mark.parametrize("mode", [synth.NORMAL, synth.DYADIC])
@pytest.mark.parametrize("router", ROUTERS)
def test_route_c1_all_tokens(mode, router):
    w = _dims("C1", router=router)
    inp = make_inputs(w.dims, w.L, w.seed, mode)
    idx, gate, score = om.route(w.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    orc, rows = _oracle_route(w.dims, w.seed, np.arange(w.L), mode)
    r = compare_routing(idx.cpu().numpy(), gate.cpu().numpy(), orc, rows, w.dims.n_rows, w.dims.n_cols)
    assert r["mismatch"] == 0, r
    assert r["gate_err"] <= 1e-5
    # ordering: sorted by (key desc, id asc) exactly like the oracle
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(-1, w.dims.top_k), orc["idx"])
    np.testing.assert_allclose(score.cpu().numpy().reshape(-1, w.dims.top_k), orc["score"], atol=1e-4)
    np.testing.assert_allclose(gate.sum(-1).cpu().numpy(), 1.0, atol=1e-6)


@pytest.mark.parametrize("name,L", [("C1", 256), ("C2", 512), ("C3a", 128), ("C4", 64)])
@pytest.mark.parametrize("mode", [synth.NORMAL, synth.DYADIC])
@pytest.mark.parametrize("method", [om.LOGITS_ROUTE, om.LOGITS_EXACT_F64])
def test_logits_bitwise_exact(name, L, mode, method):
    """Q9: every logit is RN32 of the exact dot product -- bit-identical to the oracle."""
    w = _dims(name)
    inp = make_inputs(w.dims, L, w.seed, mode, skip=("W", "V", "w_gate_up", "w_down"))
    lg = om.router_logits(w.dims, inp["x"], inp["subkeys"], method=method)
    torch.cuda.synchronize()
    x = host_rows(w.dims, w.seed, "x", np.arange(L), mode)
    sub = host_rows(w.dims, w.seed, "subkeys", None, mode).reshape(w.dims.n_heads, -1, w.dims.d)
    want = oracle.logits(x, sub)
    got = lg.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), np.argwhere(got != want)[:5]


def test_logits_fallback_rows_bitwise():
    """Rows whose exponents span more than 22 bits cannot be written as three int8
    digits; the library recomputes them with the fp64 path -- still exact."""
    d = om.LayerDims(d=64, n_rows=16, n_cols=16, top_k=4)
    L = 40
    inp = make_inputs(d, L, 7, skip=("W", "V"))
    x, sub = inp["x"].clone(), inp["subkeys"].clone()
    x[3, 5] = 2.0 ** 12   # token 3 spans 2^12 .. 2^-15
    x[17, 0] = 2.0 ** -40
    sub[0, 9, 1] = 2.0 ** 9  # sub-key row 9 spans 2^9 .. 2^-21
    lg = om.router_logits(d, x, sub)
    torch.cuda.synchronize()
    dec = lambda t: t.float().cpu().numpy().astype(np.float64)
    want = oracle.logits(dec(x), dec(sub))
    assert np.array_equal(lg.cpu().numpy().view(np.uint32), want.view(np.uint32))
    idx, gate, _ = om.route(d, x, sub)
    torch.cuda.synchronize()
    r = oracle.route(want.reshape(L, -1), 16, 16, 4, method=oracle.BRUTE)
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(L, 4), r["idx"])


@pytest.mark.parametrize("h,flag_sub", [(1, False), (2, False), (2, True)])
def test_route_fused_flags(h, flag_sub):
    """N4 (small K: per-half top-k' in the exact-logit GEMM epilogue; K >= 8 and enough
    (token block, half) units): tokens whose rows take the fp64 path are routed from their
    recomputed logits, every other token from the epilogue's lists; a flagged sub-key row
    sends every token through the logits -- ids, gates and scores equal the oracle."""
    d = om.LayerDims(d=64, n_rows=16, n_cols=24, top_k=8, n_heads=h)
    L = 6477  # a partial last 128-token block
    inp = make_inputs(d, L, 11, skip=("W", "V"))
    x, sub = inp["x"].clone(), inp["subkeys"].clone()
    x[3, 5] = 2.0 ** 12   # token 3 spans 2^12 .. 2^-15: fp64 path
    x[17, 0] = 2.0 ** -40
    x[L - 1, 2] = 2.0 ** 13
    if flag_sub:
        sub[h - 1, 9, 1] = 2.0 ** 9
    idx, gate, score = om.route(d, x, sub)
    torch.cuda.synchronize()
    dec = lambda t: t.float().cpu().numpy().astype(np.float64)
    lg = oracle.logits(dec(x), dec(sub)).reshape(L * h, -1)
    r = oracle.route(lg, 16, 24, 8, method=oracle.PRODUCT)
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(L * h, 8), r["idx"])
    np.testing.assert_allclose(gate.cpu().numpy().reshape(L * h, 8), r["gate"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(score.cpu().numpy().reshape(L * h, 8), r["score"], atol=1e-4, rtol=0)
    bf = oracle.route(lg[:300], 16, 24, 8, method=oracle.BRUTE)
    np.testing.assert_array_equal(r["idx"][:300], bf["idx"])


@pytest.mark.parametrize("name,L,n_check", [("C3b", 8192, 192), ("C5s", 6656, 96), ("C2", 8192, 256)])
def test_route_fused_full_configs(name, L, n_check):
    """N4 at the small-K workloads' shapes with the fused path on (enough tokens): the ids,
    gates and scores of tokens spread over the batch equal the oracle's."""
    w = _dims(name)
    inp = make_inputs(w.dims, L, w.seed, skip=("W", "V", "w_gate_up", "w_down"))
    idx, gate, score = om.route(w.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    toks = np.linspace(0, L - 1, n_check).astype(np.int64)
    orc, rows = _oracle_route(w.dims, w.seed, toks, method=oracle.PRODUCT)
    h, K = w.dims.n_heads, w.dims.top_k
    th = (toks[:, None] * h + np.arange(h)[None, :]).reshape(-1)
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(-1, K)[th], orc["idx"])
    np.testing.assert_allclose(gate.cpu().numpy().reshape(-1, K)[th], orc["gate"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(score.cpu().numpy().reshape(-1, K)[th], orc["score"], atol=1e-4, rtol=0)


def test_bf16_fast_logits_are_not_exact():
    """Why Q9 needs the exact path: fp32-accumulated tcgen05 logits differ from the
    exact ones."""
    w = _dims("C3a")
    inp = make_inputs(w.dims, 256, w.seed, skip=("W", "V", "w_gate_up", "w_down"))
    fast = om.router_logits(w.dims, inp["x"], inp["subkeys"], method=om.LOGITS_BF16_FAST)
    exact = om.router_logits(w.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    err = (fast.double() - exact.double()).abs().max().item()
    assert 0 < err < 1e-3


@pytest.mark.parametrize("router", ROUTERS)
def test_route_c2_multihead(router):
    w = _dims("C2", router=router)
    L = 1024
    inp = make_inputs(w.dims, L, w.seed, skip=("W", "V"))
    idx, gate, _ = om.route(w.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    orc, rows = _oracle_route(w.dims, w.seed, np.arange(L), method=oracle.PRODUCT)
    r = compare_routing(idx.cpu().numpy(), gate.cpu().numpy(), orc, rows, w.dims.n_rows, w.dims.n_cols)
    assert r["mismatch"] == 0, r
    assert r["gate_err"] <= 1e-5
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(-1, w.dims.top_k), orc["idx"])
    # brute force on a subsample pins the product path at this size too
    bf = oracle.route(rows[:64], w.dims.n_rows, w.dims.n_cols, w.dims.top_k, method=oracle.BRUTE)
    np.testing.assert_array_equal(orc["idx"][:64], bf["idx"])


@pytest.mark.parametrize("name,L", [("C3a", 96), ("C3b", 256), ("C4", 24), ("C4pp", 64), ("C5", 32), ("C5s", 64)])
def test_route_large_configs_sampled(name, L):
    """Full-size router shapes (large K, candidates in the thousands) on a token sample."""
    w = _dims(name)
    inp = make_inputs(w.dims, L, w.seed, skip=("W", "V", "w_gate_up", "w_down"))
    idx, gate, score = om.route(w.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    orc, rows = _oracle_route(w.dims, w.seed, np.arange(L), method=oracle.PRODUCT)
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(-1, w.dims.top_k), orc["idx"])
    np.testing.assert_allclose(gate.cpu().numpy().reshape(-1, w.dims.top_k), orc["gate"], atol=1e-5, rtol=0)
    np.testing.assert_allclose(score.cpu().numpy().reshape(-1, w.dims.top_k), orc["score"], atol=1e-4, rtol=0)


def test_route_batch_independent():
    """Routing of a token does not depend on the batch it is in."""
    w = _dims("C2")
    inp = make_inputs(w.dims, 300, w.seed, skip=("W", "V"))
    a, ga, _ = om.route(w.dims, inp["x"], inp["subkeys"])
    b, gb, _ = om.route(w.dims, inp["x"][100:137].contiguous(), inp["subkeys"])
    torch.cuda.synchronize()
    assert torch.equal(a[100:137], b) and torch.equal(ga[100:137], gb)


def test_route_degenerate_zero_input():
    w = _dims("C1")
    x = torch.zeros(3, w.dims.d, dtype=torch.bfloat16, device="cuda")
    inp = make_inputs(w.dims, 3, w.seed, skip=("W", "V", "w_gate_up", "w_down", "x"))
    idx, gate, _ = om.route(w.dims, x, inp["subkeys"])
    torch.cuda.synchronize()
    assert (idx.cpu().numpy() == np.arange(w.dims.top_k)).all()
    np.testing.assert_allclose(gate.cpu().numpy(), 1.0 / w.dims.top_k, atol=1e-7)


def test_route_k_equals_n():
    d = om.LayerDims(d=16, n_rows=3, n_cols=4, top_k=12, d_ff=0)
    inp = make_inputs(d, 9, 4)
    idx, gate, _ = om.route(d, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    orc, rows = _oracle_route(d, 4, np.arange(9))
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(9, 12), orc["idx"])


# ---------------------------------------------------------------- schedule
def _check_plan(plan, ids, gates, toks, b, e, B, tpb=0):
    p = oracle.schedule(ids, gates, toks, b, e, B=B, tpb=tpb)
    m = int(p["offsets"][-1])
    np.testing.assert_array_equal(plan["expert_offsets"].cpu().numpy(), p["offsets"])
    np.testing.assert_array_equal(plan["sorted_token"].cpu().numpy()[:m], p["sorted_token"])
    np.testing.assert_array_equal(plan["sorted_gate"].cpu().numpy()[:m].astype(np.float64), p["sorted_gate"])
    np.testing.assert_array_equal(plan["sorted_expert"].cpu().numpy()[:m], p["sorted_expert"])
    na = int(plan["n_active"].item())
    assert na == p["n_active"]
    np.testing.assert_array_equal(plan["active"].cpu().numpy()[:na], p["active"])
    if B > 1:
        nr = int(plan["n_runs"].item())
        assert nr == p["n_runs"]
        np.testing.assert_array_equal(plan["run_offsets"].cpu().numpy()[:nr], p["run_offsets"])


@pytest.mark.parametrize("B,Tb", [(1, 1), (2, 1), (1024, 1), (1024, 3)])
@pytest.mark.parametrize("N,L,HK,b,e", [(1024, 256, 8, 0, 1024), (65536, 2048, 64, 0, 65536),
                                        (1 << 20, 4096, 512, 0, 1 << 20), (1000, 300, 7, 250, 700),
                                        (5, 50, 3, 0, 5), (1 << 20, 16, 16, 1 << 19, 1 << 20)])
def test_schedule_bit_exact(N, L, HK, b, e, B, Tb):
    rng = np.random.default_rng(N + L)
    ids = rng.integers(0, N, (L, HK)).astype(np.int32)
    gates = rng.random((L, HK)).astype(np.float32)
    d = om.LayerDims(d=8, n_rows=N, n_cols=1, top_k=HK, d_ff=0, group_size=B, token_blocks=Tb)
    assert om.group_size(d) == B
    Tb = om.token_blocks(d, L)
    tpb = HK * -(-L // min(Tb, L)) if Tb > 1 else 0
    idx_t = torch.from_numpy(ids).cuda()
    g_t = torch.from_numpy(gates).cuda()
    plan = om.schedule(d, idx_t.reshape(-1), g_t.reshape(-1), expert_begin=b, expert_end=e)
    torch.cuda.synchronize()
    _check_plan(plan, ids.reshape(-1), gates.reshape(-1).astype(np.float64),
                np.repeat(np.arange(L), HK).astype(np.int32), b, e, B, tpb)


def test_schedule_rejects_key_overflow():
    """(token block, group) keys are uint32: token_blocks x ceil(n_loc / B) must stay
    below 2^32 - 1 or the call fails before launching anything."""
    L, N = 16384, 1 << 20
    d = om.LayerDims(d=8, n_rows=N, n_cols=1, top_k=1, d_ff=0, group_size=2, token_blocks=L)
    ids = torch.zeros(L, dtype=torch.int32, device="cuda")
    with pytest.raises(om.OmniMoEError, match="SHAPE"):
        om.schedule(d, ids, torch.ones(L, device="cuda"))
    d2 = om.LayerDims(d=8, n_rows=N, n_cols=1, top_k=1, d_ff=0, group_size=2, token_blocks=4096)
    om.schedule(d2, ids, torch.ones(L, device="cuda"))  # 4096 x 2^19 = 2^31: fits


@pytest.mark.parametrize("B", [1, 64])
def test_schedule_all_same_expert_and_empty(B):
    d = om.LayerDims(d=8, n_rows=64, n_cols=64, top_k=4, d_ff=0, group_size=B)
    ids = np.full(40000, 17, np.int32)
    gates = np.linspace(0, 1, 40000).astype(np.float32)
    plan = om.schedule(d, torch.from_numpy(ids).cuda(), torch.from_numpy(gates).cuda())
    torch.cuda.synchronize()
    _check_plan(plan, ids, gates.astype(np.float64), (np.arange(40000) // 4).astype(np.int32), 0, 4096, B)
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    plan = om.schedule(d, e, torch.empty(0, device="cuda"))
    torch.cuda.synchronize()
    assert plan["n_active"].item() == 0 and plan["expert_offsets"].cpu().numpy().max() == 0
    assert plan["n_runs"].item() == 0


# ---------------------------------------------------------------- expert compute
@pytest.mark.parametrize("B", [1, 2, 512, -512])
@pytest.mark.parametrize("dtype", [om.BF16, om.F32])
@pytest.mark.parametrize("d,act", [(64, om.SILU), (72, om.SILU), (1024, om.SILU), (2048, om.SILU), (64, om.IDENTITY)])
def test_expert_fwd_given_plan(dtype, d, act, B):
    rng = np.random.default_rng(d)
    L, N, HK = 200, 3000, 12
    # B < 0: group size |B| scheduled in 3 token blocks
    dims = om.LayerDims(d=d, n_rows=N, n_cols=1, top_k=HK, d_ff=0, dtype=dtype, act=act, group_size=abs(B),
                        token_blocks=3 if B < 0 else 0)
    inp = make_inputs(dims, L, 9, skip=("subkeys",))
    # clustered ids (several tasks of a token share a group) plus repeats across tokens
    base = rng.integers(0, N - 64, L)
    ids = np.stack([b0 + rng.choice(64, HK, replace=False) for b0 in base]).astype(np.int32)
    gates = rng.random((L, HK)).astype(np.float32)
    plan = om.schedule(dims, torch.from_numpy(ids).cuda().reshape(-1), torch.from_numpy(gates).cuda().reshape(-1))
    y = om.expert_fwd(dims, inp["x"], inp["W"], inp["V"], plan)
    torch.cuda.synchronize()
    if abs(B) > 1:
        assert plan["n_runs"].item() < L * HK  # runs really merge tasks
    used = np.unique(ids)
    remap = np.searchsorted(used, ids)
    x = host_rows(dims, 9, "x", np.arange(L))
    W = host_rows(dims, 9, "W", used)
    V = host_rows(dims, 9, "V", used)
    ref = oracle.routed_token_centric(x, W, V, remap, gates.astype(np.float64), act)
    e_tok, e_elt = rel_errors(y.cpu().numpy(), ref)
    tol = 1e-5 if dtype == om.F32 else 1e-2
    assert e_tok <= tol and e_elt <= tol, (e_tok, e_elt)


# ---------------------------------------------------------------- shared MLP
@pytest.mark.parametrize("dtype", [om.BF16, om.F32])
@pytest.mark.parametrize("L,d,dff", [(256, 64, 128), (300, 1024, 1024), (130, 256, 72), (2048, 2048, 2048)])
def test_shared_mlp(dtype, L, d, dff):
    dims = om.LayerDims(d=d, n_rows=2, n_cols=2, top_k=1, d_ff=dff, dtype=dtype)
    inp = make_inputs(dims, L, 11, skip=("subkeys", "W", "V"))
    yr = torch.randn(L, d, device="cuda")
    y = om.shared_mlp(dims, inp["x"], inp["w_gate_up"], inp["w_down"], y_routed=yr)
    torch.cuda.synchronize()
    x = host_rows(dims, 11, "x", np.arange(L))
    ref = oracle.shared_mlp(x, host_rows(dims, 11, "w_gate_up"), host_rows(dims, 11, "w_down")) + yr.cpu().double().numpy()
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), ref)
    tol = 1e-5 if dtype == om.F32 else 1e-2
    assert e_tok <= tol and e_elt <= tol, (e_tok, e_elt)
    if dtype == om.BF16 and dff % 64 == 0:
        # H enters GEMM-2 as a bf16 hi + lo pair: what is left is y's own bf16 rounding
        # (<= 2^-8 relative) plus fp32 accumulation
        assert e_elt <= 4.5e-3, e_elt


# ---------------------------------------------------------------- whole layer
@pytest.mark.parametrize("dtype,mode,router", [(om.BF16, synth.NORMAL, om.ROUTER_EXACT),
                                               (om.BF16, synth.NORMAL, om.ROUTER_EXACT_F64),
                                               (om.BF16, synth.DYADIC, om.ROUTER_EXACT),
                                               (om.F32, synth.NORMAL, om.ROUTER_EXACT),
                                               (om.F32, synth.DYADIC, om.ROUTER_EXACT)])
@pytest.mark.parametrize("B", [0, 1, 5])
def test_layer_c1(dtype, mode, router, B):
    w = _dims("C1", dtype=dtype, router=router, group_size=B)
    dims = w.dims
    inp = make_inputs(dims, w.L, w.seed, mode)
    y, idx, gate = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"],
                                inp["w_down"], return_routing=True)
    torch.cuda.synchronize()
    hr = lambda n, r=None: host_rows(dims, w.seed, n, r, mode)
    ref = oracle.layer(hr("x", np.arange(w.L)), hr("subkeys").reshape(1, -1, dims.d), hr("W"), hr("V"),
                       dims.n_rows, dims.n_cols, dims.top_k, hr("w_gate_up"), hr("w_down"))
    assert np.array_equal(np.sort(idx.cpu().numpy(), -1), np.sort(ref["idx"], -1))
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), ref["y"])
    tol = 1e-5 if dtype == om.F32 else 1e-2
    assert e_tok <= tol and e_elt <= tol, (e_tok, e_elt)


def test_layer_no_shared_mlp_and_empty():
    w = _dims("C1", d_ff=0)
    inp = make_inputs(w.dims, 64, w.seed)
    y = om.layer_fwd(w.dims, inp["x"], inp["subkeys"], inp["W"], inp["V"])
    torch.cuda.synchronize()
    hr = lambda n, r=None: host_rows(w.dims, w.seed, n, r)
    ref = oracle.layer(hr("x", np.arange(64)), hr("subkeys").reshape(1, -1, w.dims.d), hr("W"), hr("V"),
                       w.dims.n_rows, w.dims.n_cols, w.dims.top_k)
    e_tok, _ = rel_errors(y.float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2
    y0 = om.layer_fwd(w.dims, inp["x"][:0], inp["subkeys"], inp["W"], inp["V"])
    assert y0.shape == (0, w.dims.d)


def test_errors_are_loud():
    w = _dims("C1")
    inp = make_inputs(w.dims, 8, w.seed)
    bad = om.LayerDims(d=64, n_rows=4, n_cols=4, top_k=17)
    with pytest.raises(om.OmniMoEError, match="SHAPE"):
        om.route(bad, inp["x"], torch.empty(1 * 8 * 64, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(om.OmniMoEError):
        om.route(w.dims, inp["x"].cpu(), inp["subkeys"])


# ---------------------------------------------------------------- full-size, sampled
@pytest.mark.parametrize("name", ["C3a", "C3b"])
def test_layer_full_size_sampled(name):
    """The bench workload at full size, in the bench's launch configuration
    (one omnimoe_layer_fwd over all L tokens); the oracle recomputes sampled
    tokens one by one (regenerating only the expert rows they select)."""
    w = _dims(name)
    dims = w.dims
    inp = make_inputs(dims, w.L, w.seed)
    y, idx, gate = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"],
                                inp["w_down"], return_routing=True)
    torch.cuda.synchronize()
    toks = np.array([0, 1, 777, 4096, 9999, w.L - 2, w.L - 1])
    hr = lambda n, r=None: host_rows(dims, w.seed, n, r)
    x = hr("x", toks)
    sub = hr("subkeys").reshape(dims.n_heads, -1, dims.d)
    lg = oracle.logits(x, sub)
    r = oracle.route(lg.reshape(len(toks) * dims.n_heads, -1), dims.n_rows, dims.n_cols, dims.top_k)
    np.testing.assert_array_equal(np.sort(idx[toks].cpu().numpy().reshape(-1, dims.top_k), -1),
                                  np.sort(r["idx"], -1))  # the layer's ids are in candidate order
    used = np.unique(r["idx"])
    idm = np.stack([used, np.arange(len(used))], 1)
    ref = oracle.layer(x, sub, hr("W", used), hr("V", used), dims.n_rows, dims.n_cols, dims.top_k,
                       hr("w_gate_up"), hr("w_down"), id_map=idm)
    e_tok, e_elt = rel_errors(y[toks].float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


# ---------------------------------------------------------------- ablation executors (N1)
@pytest.mark.parametrize("ek", [om.EXPERT_TOKEN, om.EXPERT_WARP])
def test_layer_ablation_executors(ek):
    """'w/o ECS' token-centric executor and the expert-major B = 1 plan give
    the same layer as the default grouped path and as the oracle."""
    dims = om.LayerDims(d=256, n_rows=64, n_cols=64, top_k=32, n_heads=2, d_ff=256, expert_kernel=ek,
                        group_size=1 if ek == om.EXPERT_WARP else 0)
    L = 300
    inp = make_inputs(dims, L, 13)
    y = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"], inp["w_down"])
    d0 = om.LayerDims(d=256, n_rows=64, n_cols=64, top_k=32, n_heads=2, d_ff=256)
    y0 = om.layer_fwd(d0, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"], inp["w_down"])
    torch.cuda.synchronize()
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), y0.float().cpu().numpy())
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)
    hr = lambda n, r=None: host_rows(dims, 13, n, r)
    ref = oracle.layer(hr("x", np.arange(L)), hr("subkeys").reshape(2, -1, 256), hr("W"), hr("V"), 64, 64, 32,
                       hr("w_gate_up"), hr("w_down"))
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


# ---------------------------------------------------------------- SLICED executor (V_SLICED layout)
def test_pack_v_is_a_pure_relayout():
    dims = om.LayerDims(d=2048, n_rows=37, n_cols=11, top_k=4, v_layout=om.V_SLICED)
    inp = make_inputs(dims, 1, 5, skip=("x", "subkeys", "W"))
    Vs = om.pack_v(dims, inp["V"])
    torch.cuda.synchronize()
    want = inp["V"].view(dims.N, dims.d // 64, 64).permute(1, 0, 2).contiguous()  # test-side re-layout
    assert torch.equal(Vs.view(torch.int16), want.view(torch.int16))


@pytest.fixture(params=[{}, {"v_band_bytes": 16 << 10}], ids=["bands_default", "bands_16KB"])
def v_geom(request):
    """Pass-V bands (dims.v_band_bytes): the library's choice (one band at these sizes)
    or 16 KB bands (several)."""
    return request.param


@pytest.mark.parametrize("B", [0, 2, 512])
@pytest.mark.parametrize("d,act", [(64, om.SILU), (192, om.SILU), (1024, om.SILU), (2048, om.SILU),
                                   (64, om.IDENTITY)])
@pytest.mark.parametrize("accumulate", [False, True])
@pytest.mark.parametrize("HK", [12, 96])  # pass V: 8 tokens per warp (h*K <= 64) / one token per warp
def test_expert_fwd_sliced_given_plan(d, act, B, accumulate, v_geom, HK):
    rng = np.random.default_rng(d + B)
    L, N = 200, 3000
    dims = om.LayerDims(d=d, n_rows=N, n_cols=1, top_k=HK, d_ff=0, act=act, group_size=B, v_layout=om.V_SLICED,
                        **v_geom)
    inp = make_inputs(dims, L, 9, skip=("subkeys",))
    base = rng.integers(0, N - 128, L)
    ids = np.stack([b0 + rng.choice(128, HK, replace=False) for b0 in base]).astype(np.int32)
    ids[7] = ids[3]  # two tokens with identical expert lists
    gates = rng.random((L, HK)).astype(np.float32)
    plan = om.schedule(dims, torch.from_numpy(ids).cuda().reshape(-1), torch.from_numpy(gates).cuda().reshape(-1))
    want = -(-(N * 128) // v_geom["v_band_bytes"]) if v_geom else 1
    assert om.v_bands(dims, N, L) == want
    Vs = om.pack_v(dims, inp["V"])
    y0 = torch.randn(L, d, device="cuda") if accumulate else None
    y = om.expert_fwd(dims, inp["x"], inp["W"], Vs, plan, y_routed=None if y0 is None else y0.clone(),
                      accumulate=accumulate)
    torch.cuda.synchronize()
    used = np.unique(ids)
    remap = np.searchsorted(used, ids)
    x = host_rows(dims, 9, "x", np.arange(L))
    ref = oracle.routed_token_centric(x, host_rows(dims, 9, "W", used), host_rows(dims, 9, "V", used), remap,
                                      gates.astype(np.float64), act)
    if accumulate:
        ref = ref + y0.cpu().double().numpy()
    e_tok, e_elt = rel_errors(y.cpu().numpy(), ref)
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


def test_expert_fwd_sliced_shard_and_empty_tokens(v_geom):
    """Expert range of a shard (tasks outside it are skipped) and tokens with no
    tasks in range (their y_routed rows are written as zeros)."""
    rng = np.random.default_rng(3)
    L, N, HK, b, e = 150, 4096, 8, 1024, 2048
    dims = om.LayerDims(d=256, n_rows=N, n_cols=1, top_k=HK, d_ff=0, group_size=64, v_layout=om.V_SLICED, **v_geom)
    inp = make_inputs(dims, L, 4, skip=("subkeys",))
    ids = rng.integers(0, N, (L, HK)).astype(np.int32)
    ids[10] = rng.integers(3000, N, HK)  # token 10: nothing in [b, e)
    gates = rng.random((L, HK)).astype(np.float32)
    plan = om.schedule(dims, torch.from_numpy(ids).cuda().reshape(-1), torch.from_numpy(gates).cuda().reshape(-1),
                       expert_begin=b, expert_end=e)
    Vs = om.pack_v(dims, inp["V"][b:e].contiguous())
    y = om.expert_fwd(dims, inp["x"], inp["W"][b:e].contiguous(), Vs, plan)
    torch.cuda.synchronize()
    x = host_rows(dims, 4, "x", np.arange(L))
    mask = (ids >= b) & (ids < e)
    used = np.arange(b, e)
    remap = np.where(mask, ids - b, 0)
    g = np.where(mask, gates, 0).astype(np.float64)
    ref = oracle.routed_token_centric(x, host_rows(dims, 4, "W", used), host_rows(dims, 4, "V", used), remap, g)
    assert np.all(y[10].cpu().numpy() == 0)
    e_tok, e_elt = rel_errors(np.delete(y.cpu().numpy(), 10, 0), np.delete(ref, 10, 0))
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


@pytest.mark.parametrize("mode", [synth.NORMAL, synth.DYADIC])
@pytest.mark.parametrize("B", [0, 5])
def test_layer_c1_sliced(mode, B, v_geom):
    w = _dims("C1", group_size=B, v_layout=om.V_SLICED, **v_geom)
    dims = w.dims
    inp = make_inputs(dims, w.L, w.seed, mode)
    Vs = om.pack_v(dims, inp["V"])
    y, idx, gate = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], Vs, inp["w_gate_up"], inp["w_down"],
                                return_routing=True)
    y2 = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], Vs, inp["w_gate_up"], inp["w_down"])
    torch.cuda.synchronize()
    assert torch.equal(y, y2)  # no atomics on the SLICED path: bitwise deterministic
    hr = lambda n, r=None: host_rows(dims, w.seed, n, r, mode)
    ref = oracle.layer(hr("x", np.arange(w.L)), hr("subkeys").reshape(1, -1, dims.d), hr("W"), hr("V"),
                       dims.n_rows, dims.n_cols, dims.top_k, hr("w_gate_up"), hr("w_down"))
    assert np.array_equal(np.sort(idx.cpu().numpy(), -1), np.sort(ref["idx"], -1))
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


@pytest.mark.parametrize("name", ["C3a", "C3b", "C4"])
def test_layer_full_size_sampled_sliced(name):
    """The bench configuration (V in the SLICED layout) at full size; sampled
    tokens recomputed by the oracle."""
    w = _dims(name, v_layout=om.V_SLICED)
    dims = w.dims
    inp = make_inputs(dims, w.L, w.seed)
    inp["V"] = om.pack_v(dims, inp["V"])
    y, idx, gate = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"],
                                inp["w_down"], return_routing=True)
    torch.cuda.synchronize()
    toks = np.array([0, 1, 777, w.L // 2 + 3, w.L - 2, w.L - 1])
    hr = lambda n, r=None: host_rows(dims, w.seed, n, r)
    x = hr("x", toks)
    sub = hr("subkeys").reshape(dims.n_heads, -1, dims.d)
    lg = oracle.logits(x, sub)
    r = oracle.route(lg.reshape(len(toks) * dims.n_heads, -1), dims.n_rows, dims.n_cols, dims.top_k)
    np.testing.assert_array_equal(np.sort(idx[toks].cpu().numpy().reshape(-1, dims.top_k), -1),
                                  np.sort(r["idx"], -1))
    used = np.unique(r["idx"])
    idm = np.stack([used, np.arange(len(used))], 1)
    ref = oracle.layer(x, sub, hr("W", used), hr("V", used), dims.n_rows, dims.n_cols, dims.top_k,
                       hr("w_gate_up"), hr("w_down"), id_map=idm)
    e_tok, e_elt = rel_errors(y[toks].float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


def test_sliced_layout_errors():
    with pytest.raises(om.OmniMoEError, match="UNSUPPORTED"):
        om.workspace_size(om.LayerDims(d=64, n_rows=4, n_cols=4, top_k=2, dtype=om.F32, v_layout=om.V_SLICED), 8,
                          om.WS_LAYER)
    with pytest.raises(om.OmniMoEError, match="INVALID_ARGUMENT"):
        om.workspace_size(om.LayerDims(d=64, n_rows=4, n_cols=4, top_k=2, expert_kernel=om.EXPERT_SLICED), 8,
                          om.WS_LAYER)
    with pytest.raises(om.OmniMoEError, match="UNSUPPORTED"):  # 64-column slices: d % 64 == 0
        om.workspace_size(om.LayerDims(d=96, n_rows=4, n_cols=4, top_k=2, v_layout=om.V_SLICED), 8, om.WS_LAYER)


@pytest.mark.parametrize("name,L", [("C1", 256), ("C3a", 64), ("C4", 16), ("C4pp", 48), ("C5", 48)])
def test_route_candidate_order(name, L):
    """ORDER_CANDIDATE (the layer's routing, warp bucket selection): same id sets and
    gates as the key-ordered route, ids in Cartesian candidate order."""
    w = _dims(name)
    wc = _dims(name, route_order=om.ORDER_CANDIDATE)
    inp = make_inputs(w.dims, L, w.seed, skip=("W", "V", "w_gate_up", "w_down"))
    a, ga, sa = om.route(w.dims, inp["x"], inp["subkeys"])
    b, gb, sb = om.route(wc.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    K = w.dims.top_k
    a, b = a.cpu().numpy().reshape(-1, K), b.cpu().numpy().reshape(-1, K)
    oa, ob = np.argsort(a, -1), np.argsort(b, -1)
    np.testing.assert_array_equal(np.take_along_axis(a, oa, -1), np.take_along_axis(b, ob, -1))
    # scores = key - lse_r - lse_c: the two kernels sum a half's exp terms in different
    # orders (fp32, 2048 terms at C5), so scores get the oracle protocol's 1e-4
    # (1e-6 wherever the halves are at most 1024 keys, which holds for all but C5)
    stol = 1e-4 if name == "C5" else 1e-6
    for x_, y_, tol in [(ga, gb, 1e-6), (sa, sb, stol)]:
        x_, y_ = x_.cpu().numpy().reshape(-1, K), y_.cpu().numpy().reshape(-1, K)
        np.testing.assert_allclose(np.take_along_axis(x_, oa, -1), np.take_along_axis(y_, ob, -1), atol=tol)


@pytest.mark.parametrize("nr,nc,K", [(2500, 1100, 100), (3000, 37, 40), (1025, 4096, 700)])
def test_route_candidate_order_long_halves(nr, nc, K):
    """The warp bucket selection on halves longer than 1024 keys (C5's 2048 x 2048 grid and
    ragged shapes): candidate-order ids are the oracle's set, gates match."""
    dims = om.LayerDims(d=128, n_rows=nr, n_cols=nc, top_k=K, d_ff=0, route_order=om.ORDER_CANDIDATE)
    L, seed = 40, 7
    inp = make_inputs(dims, L, seed, skip=("W", "V", "w_gate_up", "w_down"))
    idx, gate, _ = om.route(dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    r, _rows = _oracle_route(dims, seed, np.arange(L), method=oracle.PRODUCT)
    got = idx.cpu().numpy().reshape(L, K)
    o = np.argsort(got, -1)
    ref_o = np.argsort(r["idx"], -1)
    np.testing.assert_array_equal(np.take_along_axis(got, o, -1), np.take_along_axis(r["idx"], ref_o, -1))
    np.testing.assert_allclose(np.take_along_axis(gate.cpu().numpy().reshape(L, K), o, -1),
                               np.take_along_axis(r["gate"], ref_o, -1), atol=1e-5, rtol=0)


# ---------------------------------------------------------------- N1: load metrics
@pytest.mark.parametrize("N,M,skew", [(1024, 2048, 0.0), (1 << 20, 1 << 20, 0.0), (4096, 50000, 2.0)])
def test_load_stats_match_oracle(N, M, skew):
    rng = np.random.default_rng(N + M)
    p = rng.random(N) ** (1 + 8 * skew)
    ids = rng.choice(N, M, p=p / p.sum()).astype(np.int32)
    d = om.LayerDims(d=8, n_rows=N, n_cols=1, top_k=1, d_ff=0, group_size=1)
    plan = om.schedule(d, torch.from_numpy(ids).cuda(), torch.ones(M, device="cuda"))
    got = om.load_stats(plan).cpu().numpy()
    want = oracle.load_stats(np.bincount(ids, minlength=N))
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- N1: the dense-router ablation ("w/o CPR")
@pytest.mark.parametrize("d,nr,nc,K,h,L", [(64, 32, 32, 8, 2, 200), (256, 64, 64, 100, 1, 130),
                                           (1024, 320, 320, 4096, 1, 12)])
def test_dense_router_selection_exact(d, nr, nc, K, h, L):
    """Given the GEMM's logits, the dense top-K is exact (ids in key order, gates);
    the logits themselves are the bf16 GEMM's fp32-accumulated dot products."""
    dims = om.LayerDims(d=d, n_rows=nr, n_cols=nc, top_k=K, n_heads=h, router=om.ROUTER_DENSE)
    inp = make_inputs(dims, L, 21, skip=("W", "V", "w_gate_up", "w_down"))
    idx, gate, score = om.route(dims, inp["x"], inp["subkeys"])
    lg = om.router_logits(dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    rows = lg.cpu().numpy().reshape(L * h, -1)
    ref = oracle.dense_route(rows, K)
    np.testing.assert_array_equal(idx.cpu().numpy().reshape(-1, K), ref["idx"])
    np.testing.assert_allclose(gate.cpu().numpy().reshape(-1, K), ref["gate"], atol=1e-6)
    lse = np.log(np.exp(rows.astype(np.float64) - rows.max(1, keepdims=True)).sum(1)) + rows.max(1)
    np.testing.assert_allclose(score.cpu().numpy().reshape(-1, K), ref["key"] - lse[:, None], atol=1e-4)
    # the logits against the exact dot products (an fp32-accumulated GEMM: not RN32-exact)
    x = host_rows(dims, 21, "x", np.arange(L))
    sub = host_rows(dims, 21, "subkeys").reshape(h, -1, d)
    exact = oracle.logits(x, sub).reshape(L * h, -1)
    assert np.abs(rows.astype(np.float64) - exact).max() <= 2e-5 * max(1.0, np.abs(exact).max())


def test_layer_dense_router():
    """The 'w/o CPR' layer: dense routing + the same schedule / SLICED executor /
    shared MLP, against the oracle evaluated on the GPU's routing decision."""
    dims = om.LayerDims(d=64, n_rows=32, n_cols=32, top_k=8, d_ff=128, router=om.ROUTER_DENSE, v_layout=om.V_SLICED)
    L = 256
    inp = make_inputs(dims, L, 0)
    y, idx, gate = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], om.pack_v(dims, inp["V"]),
                                inp["w_gate_up"], inp["w_down"], return_routing=True)
    torch.cuda.synchronize()
    hr = lambda n, r=None: host_rows(dims, 0, n, r)
    x = hr("x", np.arange(L))
    ids = idx.cpu().numpy().reshape(L, -1)
    ref = oracle.routed_token_centric(x, hr("W"), hr("V"), ids, gate.cpu().numpy().reshape(L, -1).astype(np.float64))
    ref += oracle.shared_mlp(x, hr("w_gate_up"), hr("w_down"))
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), ref)
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


def test_layer_low_eta_uses_token_executor():
    """AUTO + ROWS at eta < 2 (no expert shared by two tasks) runs the token-centric
    executor without a schedule; results against the oracle."""
    dims = om.LayerDims(d=256, n_rows=64, n_cols=64, top_k=2, d_ff=256)
    L = 200
    assert om.layer_executor(dims, L) == om.EXPERT_TOKEN
    assert om.layer_executor(om.LayerDims(d=256, n_rows=64, n_cols=64, top_k=64, d_ff=256), L) == om.EXPERT_GROUP
    inp = make_inputs(dims, L, 17)
    y = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"], inp["w_down"])
    torch.cuda.synchronize()
    hr = lambda n, r=None: host_rows(dims, 17, n, r)
    ref = oracle.layer(hr("x", np.arange(L)), hr("subkeys").reshape(1, -1, 256), hr("W"), hr("V"), 64, 64, 2,
                       hr("w_gate_up"), hr("w_down"))
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


# ---------------------------------------------------------------- N2: routed-branch backward
@pytest.mark.parametrize("N", [3000, 800])  # eta 1.45 (fused kernel) / 3.2 (row-gather passes when d % 512 == 0)
@pytest.mark.parametrize("d,act", [(64, om.SILU), (256, om.SILU), (1024, om.SILU), (1536, om.SILU), (2048, om.SILU),
                                   (128, om.IDENTITY), (512, om.IDENTITY)])
def test_expert_bwd_matches_oracle(d, act, N):
    rng = np.random.default_rng(d + act)
    L, HK = 200, 12
    dims = om.LayerDims(d=d, n_rows=N, n_cols=1, top_k=HK, d_ff=0, act=act, group_size=1)
    inp = make_inputs(dims, L, 9, skip=("subkeys",))
    base = rng.integers(0, N - 64, L)
    ids = np.stack([b0 + rng.choice(64, HK, replace=False) for b0 in base]).astype(np.int32)
    gates = rng.random((L, HK)).astype(np.float32)
    plan = om.schedule(dims, torch.from_numpy(ids).cuda().reshape(-1), torch.from_numpy(gates).cuda().reshape(-1))
    dy = torch.randn(L, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(d)).to(torch.bfloat16)
    sd = om.LayerDims(d=d, n_rows=N, n_cols=1, top_k=HK, d_ff=0, v_layout=om.V_SLICED)
    Ws = om.pack_v(sd, inp["W"])
    dx, dW, dV, dg = om.expert_bwd(dims, inp["x"], inp["W"], inp["V"], Ws, plan, dy)
    torch.cuda.synchronize()
    used = np.unique(ids)
    remap = np.searchsorted(used, ids)
    ref = oracle.routed_bwd(host_rows(dims, 9, "x", np.arange(L)), host_rows(dims, 9, "W", used),
                            host_rows(dims, 9, "V", used), remap, gates.astype(np.float64),
                            dy.double().cpu().numpy(), act)
    act_ids = plan["active"][:int(plan["n_active"].item())].cpu().numpy()
    np.testing.assert_array_equal(act_ids, used)
    for got, want in ((dx, ref["dx"]), (dW, ref["dW"]), (dV, ref["dV"])):
        e_tok, e_elt = rel_errors(got.cpu().numpy(), want)
        assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)
    np.testing.assert_allclose(dg.cpu().numpy(), ref["dgate"].reshape(-1),
                               atol=1e-2 * np.abs(ref["dgate"]).max(), rtol=1e-2)


def test_expert_bwd_needs_one_band():
    """dgate is written in task order through the plan's V order, which needs one band."""
    dims = om.LayerDims(d=512, n_rows=3000, n_cols=1, top_k=4, d_ff=0, group_size=1, v_band_bytes=64 << 10)
    assert om.v_bands(dims, dims.N, 8) > 1
    inp = make_inputs(dims, 8, 2, skip=("subkeys",))
    ids = torch.arange(32, dtype=torch.int32, device="cuda") * 90
    plan = om.schedule(dims, ids, torch.ones(32, device="cuda"))
    Ws = om.pack_v(om.LayerDims(d=512, n_rows=3000, n_cols=1, top_k=4, v_layout=om.V_SLICED), inp["W"])
    with pytest.raises(om.OmniMoEError, match="UNSUPPORTED"):
        om.expert_bwd(dims, inp["x"], inp["W"], inp["V"], Ws, plan, inp["x"])


@pytest.mark.parametrize("d,nr,nc,K,h,L", [(64, 32, 32, 8, 1, 256), (256, 64, 64, 64, 2, 300), (1024, 256, 256, 512, 1, 64)])
def test_router_bwd_matches_oracle(d, nr, nc, K, h, L):
    dims = om.LayerDims(d=d, n_rows=nr, n_cols=nc, top_k=K, n_heads=h, d_ff=0)
    inp = make_inputs(dims, L, 31, skip=("W", "V", "w_gate_up", "w_down"))
    idx, gate, _ = om.route(dims, inp["x"], inp["subkeys"])
    dg = torch.randn(L, h, K, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))
    dx0 = torch.randn(L, d, device="cuda")
    dx, dsub = om.router_bwd(dims, inp["x"], inp["subkeys"], idx, gate, dg, dx=dx0.clone(), accumulate_dx=True)
    torch.cuda.synchronize()
    x = host_rows(dims, 31, "x", np.arange(L))
    sub = host_rows(dims, 31, "subkeys").reshape(h, nr + nc, d)
    rdx, rdsub = oracle.router_bwd(x, sub, nr, nc, idx.cpu().numpy(), gate.cpu().double().numpy(),
                                   dg.cpu().double().numpy())
    e = rel_errors((dx - dx0).cpu().numpy(), rdx)
    assert e[0] <= 1e-2 and e[1] <= 1e-2, e
    used = np.abs(rdsub).reshape(-1, d).sum(1) > 0        # sub-key rows never selected get 0
    got = dsub.cpu().numpy().reshape(-1, d)
    assert np.all(got[~used] == 0)
    e = rel_errors(got[used], rdsub.reshape(-1, d)[used])
    assert e[0] <= 1e-2 and e[1] <= 1e-2, e


@pytest.mark.parametrize("L,d,dff", [(256, 64, 128), (300, 256, 512), (130, 1024, 1024)])
def test_shared_mlp_bwd_matches_oracle(L, d, dff):
    dims = om.LayerDims(d=d, n_rows=2, n_cols=2, top_k=1, d_ff=dff)
    inp = make_inputs(dims, L, 13, skip=("subkeys", "W", "V"))
    dy = torch.randn(L, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)).to(torch.bfloat16)
    dx, dgu, ddn = om.shared_mlp_bwd(dims, inp["x"], inp["w_gate_up"], inp["w_down"], dy)
    torch.cuda.synchronize()
    rdx, rdgu, rddn = oracle.mlp_bwd(host_rows(dims, 13, "x", np.arange(L)), host_rows(dims, 13, "w_gate_up"),
                                     host_rows(dims, 13, "w_down"), dy.double().cpu().numpy())
    for got, want in ((dx, rdx), (dgu, rdgu), (ddn, rddn)):
        e = rel_errors(got.cpu().numpy().reshape(want.shape[0], -1), want.reshape(want.shape[0], -1))
        assert e[0] <= 1e-2 and e[1] <= 1e-2, e


def test_layer_bwd_composition():
    """N2 end to end at a C1-like shape: the three backward calls against the oracle's
    routed / router / MLP backward on the GPU's own routing (dx summed over all three)."""
    w = _dims("C1", v_layout=om.V_SLICED)
    dims = w.dims
    L = w.L
    inp = make_inputs(dims, L, w.seed)
    Vs, Ws = om.pack_v(dims, inp["V"]), om.pack_v(dims, inp["W"])
    idx, gate, _ = om.route(dims, inp["x"], inp["subkeys"])
    plan = om.schedule(dims, idx.reshape(-1), gate.reshape(-1))
    dy = torch.randn(L, dims.d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5)).to(torch.bfloat16)
    g = om.layer_bwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], Ws, inp["w_gate_up"], inp["w_down"],
                     idx, gate, plan, dy)
    torch.cuda.synchronize()
    hr = lambda n, r=None: host_rows(dims, w.seed, n, r)
    x, W, V = hr("x", np.arange(L)), hr("W"), hr("V")
    ids = idx.cpu().numpy().reshape(L, -1)
    gt = gate.cpu().double().numpy().reshape(L, -1)
    dyn = dy.double().cpu().numpy()
    rb = oracle.routed_bwd(x, W, V, ids, gt, dyn)
    rdx, rdsub = oracle.router_bwd(x, hr("subkeys").reshape(1, -1, dims.d), dims.n_rows, dims.n_cols,
                                   idx.cpu().numpy(), gate.cpu().double().numpy(), rb["dgate"].reshape(L, 1, -1))
    mdx, mdgu, mddn = oracle.mlp_bwd(x, hr("w_gate_up"), hr("w_down"), dyn)
    act = g["active"].cpu().numpy()
    checks = [(g["dx"], rb["dx"] + rdx + mdx), (g["dsubkeys"].reshape(-1, dims.d), rdsub.reshape(-1, dims.d)),
              (g["dW_act"], rb["dW"][act]), (g["dV_act"], rb["dV"][act]), (g["dw_gate_up"], mdgu),
              (g["dw_down"], mddn)]
    for got, want in checks:
        got = got.cpu().numpy()
        keep = np.abs(want).sum(1) > 0
        e = rel_errors(got[keep], want[keep])
        assert e[0] <= 1e-2 and e[1] <= 1e-2, e


@pytest.mark.parametrize("name,L,chunks,vl", [("C1", 256, 1, om.V_SLICED), ("C1", 300, 3, om.V_SLICED),
                                              ("C3a", 1000, 4, om.V_SLICED), ("C3b", 777, 4, om.V_ROWS)])
def test_layer_fwd_host_equals_device_call(name, L, chunks, vl):
    """The host-buffer call (chunked, transfers overlapped) gives the device call's bits."""
    w = _dims(name, v_layout=vl)
    dims = w.dims
    inp = make_inputs(dims, L, w.seed)
    V = om.pack_v(dims, inp["V"]) if vl == om.V_SLICED else inp["V"]
    y = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], V, inp["w_gate_up"], inp["w_down"])
    xh = inp["x"].cpu().pin_memory()
    yh = om.layer_fwd_host(dims, xh, inp["subkeys"], inp["W"], V, inp["w_gate_up"], inp["w_down"], chunks=chunks)
    torch.cuda.synchronize()
    assert torch.equal(yh.view(torch.int16), y.cpu().view(torch.int16))


def test_layer_high_eta_uses_dense_executor():
    """AUTO + ROWS at eta >= 64 (one head) runs the routed branch as two tcgen05 GEMMs;
    results against the oracle on the GPU's routing decision, and the same layer with
    the grouped executor."""
    dims = om.LayerDims(d=256, n_rows=32, n_cols=32, top_k=256, d_ff=256)
    L = 1024
    assert om.layer_executor(dims, L) == om.EXPERT_DENSE
    inp = make_inputs(dims, L, 23)
    y, idx, gate = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"],
                                inp["w_down"], return_routing=True)
    g = om.LayerDims(d=256, n_rows=32, n_cols=32, top_k=256, d_ff=256, expert_kernel=om.EXPERT_GROUP, group_size=64)
    y_g = om.layer_fwd(g, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"], inp["w_down"])
    torch.cuda.synchronize()
    hr = lambda n, r=None: host_rows(dims, 23, n, r)
    x = hr("x", np.arange(L))
    ref = oracle.routed_token_centric(x, hr("W"), hr("V"), idx.cpu().numpy().reshape(L, -1),
                                      gate.cpu().double().numpy().reshape(L, -1))
    ref += oracle.shared_mlp(x, hr("w_gate_up"), hr("w_down"))
    # the routed branch alone (fp32) against the oracle: the executor's own error
    yr = om.expert_fwd_dense(dims, inp["x"], inp["W"], inp["V"], idx.reshape(L, -1), gate.reshape(L, -1))
    torch.cuda.synchronize()
    routed = oracle.routed_token_centric(x, hr("W"), hr("V"), idx.cpu().numpy().reshape(L, -1),
                                         gate.cpu().double().numpy().reshape(L, -1))
    e = rel_errors(yr.cpu().numpy(), routed)
    assert e[0] <= 1e-2 and e[1] <= 1e-2, e
    # the layers (bf16 outputs): dense vs grouped executor, and against the oracle per token
    e = rel_errors(y.float().cpu().numpy(), y_g.float().cpu().numpy())
    assert e[0] <= 1e-2 and e[1] <= 1e-2, e
    assert rel_errors(y.float().cpu().numpy(), ref)[0] <= 1e-2


def test_layer_full_size_sampled_dense_c4():
    """C4 at full size in the bench's configuration (ROWS layout -> the dense executor);
    sampled tokens recomputed by the oracle."""
    w = _dims("C4")
    dims = w.dims
    assert om.layer_executor(dims, w.L) == om.EXPERT_DENSE
    inp = make_inputs(dims, w.L, w.seed)
    y, idx, gate = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"],
                                inp["w_down"], return_routing=True)
    torch.cuda.synchronize()
    toks = np.array([0, 5, 2048, w.L - 1])
    hr = lambda n, r=None: host_rows(dims, w.seed, n, r)
    x = hr("x", toks)
    sub = hr("subkeys").reshape(dims.n_heads, -1, dims.d)
    r = oracle.route(oracle.logits(x, sub).reshape(len(toks), -1), dims.n_rows, dims.n_cols, dims.top_k)
    np.testing.assert_array_equal(np.sort(idx[toks].cpu().numpy().reshape(-1, dims.top_k), -1),
                                  np.sort(r["idx"], -1))
    used = np.unique(r["idx"])
    idm = np.stack([used, np.arange(len(used))], 1)
    ref = oracle.layer(x, sub, hr("W", used), hr("V", used), dims.n_rows, dims.n_cols, dims.top_k,
                       hr("w_gate_up"), hr("w_down"), id_map=idm)
    e = rel_errors(y[toks].float().cpu().numpy(), ref["y"])
    assert e[0] <= 1e-2 and e[1] <= 1e-2, e


@pytest.mark.parametrize("d,nr,nc,K,L,act", [
    (96, 37, 37, 5, 200, om.SILU),        # N = 1369 (not a multiple of 8, 32 or 64), d % 64 != 0
    (128, 40, 40, 800, 130, om.SILU),     # K / N = 50%: dense chunks, gates beyond the staged 16
    (64, 16, 16, 256, 257, om.IDENTITY),  # every expert selected by every token
    (256, 64, 48, 40, 1, om.SILU),        # one token
    (64, 600, 600, 64, 9, om.SILU),       # N = 360,000: rows too wide for the shared-memory prep
])
def test_expert_fwd_dense_ragged(d, nr, nc, K, L, act):
    """The dense executor (gated GEMM epilogue + MN-major V operand) on ragged shapes, from a
    seeded random routing, against the oracle's token-centric routed branch."""
    dims = om.LayerDims(d=d, n_rows=nr, n_cols=nc, top_k=K, d_ff=0, act=act)
    N = nr * nc
    inp = make_inputs(dims, L, 41)
    g = torch.Generator().manual_seed(L * 1000 + K)
    ids = torch.stack([torch.randperm(N, generator=g)[:K] for _ in range(L)]).to(torch.int32)
    gates = torch.rand((L, K), generator=g, dtype=torch.float32) + 0.05
    gates /= gates.sum(-1, keepdim=True)
    yr = om.expert_fwd_dense(dims, inp["x"], inp["W"], inp["V"], ids.cuda(), gates.cuda())
    torch.cuda.synchronize()
    hr = lambda n, r=None: host_rows(dims, 41, n, r)
    ref = oracle.routed_token_centric(hr("x", np.arange(L)), hr("W"), hr("V"), ids.numpy(),
                                      gates.double().numpy(), act=act)
    e = rel_errors(yr.cpu().numpy(), ref)
    assert e[0] <= 1e-2 and e[1] <= 1e-2, e
