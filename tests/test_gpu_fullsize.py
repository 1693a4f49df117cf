"""Full-size parity (-m gpu), in the launch configuration bench.py times.

* whole-batch routing at C3a (all 16,384 tokens) and C4 (all 4,096): every logit
  bit-identical to oracle.logits -- at C3a the persistent i8 limb GEMM walks ~19
  tiles per CTA, so its cross-tile stage ring and accumulator reuse are covered --
  and every token-head's id set (and, in key order, the ids' order) equal to
  oracle.route, with the mismatch / allowed / disallowed counts of reading Q10;
* the C5 layer (N = 2^22, 65,536 tokens, SLICED executor with its expert bands)
  on 256 tokens spread over the batch, recomputed one by one by oracle.layer;
* the all-fp32 mode at a reduced C3 (d = 2048, N = 2^20, K = 512, 256 tokens) at
  the north star's 1e-5, for every executor the fp32 layer can run (the token-centric
  one is bf16 only).

Expected values come only from oracle/ (PAPER:131-144 Eq.TopK/Eq.Gate/Eq.MoE,
PAPER:211-224 Eq.Logits/Eq.LSM, PAPER:182-186 Eq.Assemble); inputs from synth/."""
import numpy as np
import pytest
import torch

import oracle
from synth.workloads import make_inputs
from paper_2602_05711_b200 import configs, omnimoe as om
from tests.helpers import host_rows, rel_errors, routing_counts

pytestmark = pytest.mark.gpu


def _oracle_logits(dims, seed, tokens, chunk=2048):
    sub = host_rows(dims, seed, "subkeys").reshape(dims.n_heads, -1, dims.d)
    out = []
    for a in range(0, len(tokens), chunk):
        out.append(oracle.logits(host_rows(dims, seed, "x", tokens[a:a + chunk]), sub))
    return np.concatenate(out), sub


@pytest.fixture(scope="module", params=["C3a", "C4"])
def whole_batch(request):
    w = configs.get(request.param)
    dims = w.dims
    lg, sub = _oracle_logits(dims, w.seed, np.arange(w.L))
    rows = lg.reshape(-1, dims.n_rows + dims.n_cols)
    orc = oracle.route(rows, dims.n_rows, dims.n_cols, dims.top_k, method=oracle.PRODUCT)
    inp = make_inputs(dims, w.L, w.seed, skip=("W", "V", "w_gate_up", "w_down"))
    return w, lg, rows, orc, inp


def test_whole_batch_logits_bitwise(whole_batch):
    w, lg, _, _, inp = whole_batch
    got = om.router_logits(w.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    got = got.cpu().numpy().reshape(lg.shape)
    bad = np.argwhere(got.view(np.uint32) != lg.view(np.uint32))
    assert len(bad) == 0, (len(bad), bad[:5])


def test_whole_batch_routing_key_order(whole_batch):
    w, _, rows, orc, inp = whole_batch
    K = w.dims.top_k
    idx, gate, score = om.route(w.dims, inp["x"], inp["subkeys"])
    torch.cuda.synchronize()
    idx, gate, score = (t.cpu().numpy().reshape(-1, K) for t in (idx, gate, score))
    c = routing_counts(idx, gate, orc, rows, w.dims.n_rows, w.dims.n_cols)
    assert (c["mismatch"], c["allowed"], c["disallowed"]) == (0, 0, 0), c
    assert c["gate_err"] <= 1e-5, c
    np.testing.assert_array_equal(idx, orc["idx"])  # (key desc, id asc), reading Q12
    np.testing.assert_allclose(score, orc["score"], atol=1e-4, rtol=0)


def test_whole_batch_routing_layer_order(whole_batch):
    """The layer's own routing (candidate order, warp bucket selection)."""
    w, _, rows, orc, inp = whole_batch
    K = w.dims.top_k
    wc = configs.get(w.name, route_order=om.ORDER_CANDIDATE)
    idx, gate, _ = om.route(wc.dims, inp["x"], inp["subkeys"], want_score=False)
    torch.cuda.synchronize()
    c = routing_counts(idx.cpu().numpy().reshape(-1, K), gate.cpu().numpy().reshape(-1, K), orc, rows,
                       w.dims.n_rows, w.dims.n_cols)
    assert (c["mismatch"], c["allowed"], c["disallowed"]) == (0, 0, 0), c
    assert c["gate_err"] <= 1e-5, c


def _oracle_layer_chunked(dims, seed, toks, chunk=64):
    """oracle.layer on tokens `toks`, a chunk at a time, regenerating only the expert
    rows each chunk selects."""
    hr = lambda n, r=None: host_rows(dims, seed, n, r)
    sub = hr("subkeys").reshape(dims.n_heads, -1, dims.d)
    wgu, wdn = (hr("w_gate_up"), hr("w_down")) if dims.d_ff else (None, None)
    ys, ids = [], []
    for a in range(0, len(toks), chunk):
        x = hr("x", toks[a:a + chunk])
        lg = oracle.logits(x, sub)
        r = oracle.route(lg.reshape(-1, dims.n_rows + dims.n_cols), dims.n_rows, dims.n_cols, dims.top_k)
        used = np.unique(r["idx"])
        idm = np.stack([used, np.arange(len(used))], 1)
        ref = oracle.layer(x, sub, hr("W", used), hr("V", used), dims.n_rows, dims.n_cols, dims.top_k, wgu, wdn,
                           act=dims.act, id_map=idm)
        ys.append(ref["y"])
        ids.append(ref["idx"])
    return np.concatenate(ys), np.concatenate(ids)


def test_layer_c5_full_size_sliced():
    """configs[4] on one GPU (R = 1): N = 2048 x 2048, 65,536 tokens, K = 512, the
    SLICED executor with the expert bands the bench runs; 256 tokens recomputed."""
    w = configs.get("C5", v_layout=om.V_SLICED)
    dims = w.dims
    assert om.layer_executor(dims, w.L) == om.EXPERT_SLICED and om.v_bands(dims, dims.N, w.L) > 1
    inp = make_inputs(dims, w.L, w.seed)
    inp["V"] = om.pack_v(dims, inp["V"])
    torch.cuda.synchronize()
    y, idx, _ = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"],
                             inp["w_down"], return_routing=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    toks = np.unique(np.concatenate([[0, 1, w.L // 2, w.L - 2, w.L - 1], rng.choice(w.L, 251, replace=False)]))
    assert len(toks) >= 256
    y_ref, idx_ref = _oracle_layer_chunked(dims, w.seed, toks)
    got = idx[torch.from_numpy(toks).cuda()].cpu().numpy().reshape(len(toks), -1)
    np.testing.assert_array_equal(np.sort(got, -1), np.sort(idx_ref.reshape(len(toks), -1), -1))
    e_tok, e_elt = rel_errors(y[torch.from_numpy(toks).cuda()].float().cpu().numpy(), y_ref)
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


@pytest.fixture(scope="module")
def c3_f32():
    """Reduced C3 in the all-fp32 mode: d = 2048, N = 2^20, K = 512, 256 tokens."""
    w = configs.get("C3a", dtype=om.F32, L=256)
    inp = make_inputs(w.dims, w.L, w.seed)
    y_ref, idx_ref = _oracle_layer_chunked(w.dims, w.seed, np.arange(w.L))
    return w, inp, y_ref, idx_ref


@pytest.mark.parametrize("ek,B", [(om.EXPERT_AUTO, 0), (om.EXPERT_WARP, 1), (om.EXPERT_GROUP, 8192)])
def test_layer_f32_reduced_c3(c3_f32, ek, B):
    w, inp, y_ref, idx_ref = c3_f32
    dims = configs.get("C3a", dtype=om.F32, expert_kernel=ek, group_size=B).dims
    y, idx, _ = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp["w_gate_up"], inp["w_down"],
                             return_routing=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(np.sort(idx.cpu().numpy().reshape(w.L, -1), -1),
                                  np.sort(idx_ref.reshape(w.L, -1), -1))
    e_tok, e_elt = rel_errors(y.cpu().numpy(), y_ref)
    assert e_tok <= 1e-5 and e_elt <= 1e-5, (e_tok, e_elt)


@pytest.mark.parametrize("K", [1, 4, 16, 64])
@pytest.mark.parametrize("L", [1024, 2048, 4096, 8192, 16384])
def test_c2_sweep_brute_force(L, K):
    """configs[1]'s router-only sweep (tools/c2_sweep.py times it): at every (L, K) point
    the key-ordered ids of a 24-token subsample equal brute force over all N cells
    (Eq.TopK by definition), and the whole batch's sets equal the product path."""
    w = configs.get("C2", top_k=K)
    dims = w.dims
    inp = make_inputs(dims, L, w.seed, skip=("W", "V", "w_gate_up", "w_down"))
    idx, gate, _ = om.route(dims, inp["x"], inp["subkeys"], want_score=False)
    torch.cuda.synchronize()
    idx = idx.cpu().numpy().reshape(L, dims.n_heads, K)
    toks = np.unique(np.concatenate([[0, L - 1], np.random.default_rng(L + K).choice(L, 22, replace=False)]))
    lg, _ = _oracle_logits(dims, w.seed, toks)
    rows = lg.reshape(-1, dims.n_rows + dims.n_cols)
    bf = oracle.route(rows, dims.n_rows, dims.n_cols, K, method=oracle.BRUTE)
    np.testing.assert_array_equal(idx[toks].reshape(-1, K), bf["idx"])
