"""Expert-parallel layer on the GPU (-m gpu): the real kernels (pack, unpack,
schedule, expert, combine, MLP) and the real exchange protocol, with R virtual
ranks in one process (loopback) and with a one-rank NCCL group; results must
match the single-GPU layer and the oracle."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from paper_2602_05711_b200 import configs, distributed as ep, omnimoe as om
from synth.workloads import make_inputs
from tests.helpers import host_rows, rel_errors

pytestmark = pytest.mark.gpu

MID = dict(d=256, n_rows=64, n_cols=64, top_k=32, n_heads=2, d_ff=256)


def _run_loopback(dims, L, seed, R):
    full = make_inputs(dims, L, seed)
    ops = ep.LibOps(dims)
    ops.set_mlp(full["w_gate_up"], full["w_down"])
    lpr, n_per = L // R, dims.N // R
    xs = [full["x"][r * lpr:(r + 1) * lpr] for r in range(R)]
    shards = [make_inputs(dims, 1, seed, skip=("x", "subkeys", "w_gate_up", "w_down"),
                          expert_rows=(r * n_per, (r + 1) * n_per)) for r in range(R)]
    sl = dims.v_layout == om.V_SLICED
    vs = [om.pack_v(dims, s["V"]) if sl else s["V"] for s in shards]
    ys = ep.ep_layer_fwd_loopback(ops, xs, full["subkeys"], [s["W"] for s in shards], vs, n_per)
    y1 = om.layer_fwd(dims, full["x"], full["subkeys"], full["W"], om.pack_v(dims, full["V"]) if sl else full["V"],
                      full["w_gate_up"], full["w_down"])
    torch.cuda.synchronize()
    return torch.cat(ys), y1, full


def test_synth_shard_equals_rows_of_full():
    dims = om.LayerDims(d=64, n_rows=32, n_cols=32, top_k=8)
    full = make_inputs(dims, 8, 3, skip=("x", "subkeys"))
    part = make_inputs(dims, 8, 3, skip=("x", "subkeys"), expert_rows=(256, 512))
    assert torch.equal(full["W"][256:512], part["W"]) and torch.equal(full["V"][256:512], part["V"])
    xs = make_inputs(dims, 4, 3, skip=("W", "V", "subkeys"), token_begin=5)
    xf = make_inputs(dims, 9, 3, skip=("W", "V", "subkeys"))
    assert torch.equal(xs["x"], xf["x"][5:9])


@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("vl", [om.V_ROWS, om.V_SLICED])
def test_ep_loopback_c1(R, vl):
    w = configs.get("C1", v_layout=vl)
    y, y1, _ = _run_loopback(w.dims, w.L, w.seed, R)
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), y1.float().cpu().numpy())
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)
    hr = lambda n, r=None: host_rows(w.dims, w.seed, n, r)
    ref = oracle.layer(hr("x", np.arange(w.L)), hr("subkeys").reshape(1, -1, w.dims.d), hr("W"), hr("V"),
                       w.dims.n_rows, w.dims.n_cols, w.dims.top_k, hr("w_gate_up"), hr("w_down"))
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


@pytest.mark.parametrize("R,B,vl", [(2, 0, om.V_ROWS), (4, 0, om.V_ROWS), (8, 1, om.V_ROWS), (2, 0, om.V_SLICED),
                                    (8, 0, om.V_SLICED)])
def test_ep_loopback_mid(R, B, vl):
    dims = om.LayerDims(**MID, group_size=B, v_layout=vl)
    y, y1, _ = _run_loopback(dims, 512, 5, R)
    e_tok, e_elt = rel_errors(y.float().cpu().numpy(), y1.float().cpu().numpy())
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_ep_nccl_one_rank():
    """The torch.distributed driver over a real NCCL group (world size 1: the
    only size this box has) against the single-GPU layer."""
    script = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2602_05711_b200 import distributed as ep, omnimoe as om
from synth.workloads import make_inputs
from tests.helpers import rel_errors
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
dims = om.LayerDims(d=256, n_rows=64, n_cols=64, top_k=32, n_heads=2, d_ff=256)
full = make_inputs(dims, 384, 7)
ops = ep.LibOps(dims); ops.set_mlp(full["w_gate_up"], full["w_down"])
y = ep.ep_layer_fwd(ops, ep.TorchComm(), full["x"], full["subkeys"], full["W"], full["V"], dims.N)
sd = om.LayerDims(d=256, n_rows=64, n_cols=64, top_k=32, n_heads=2, d_ff=256, v_layout=om.V_SLICED)
so = ep.LibOps(sd); so.set_mlp(full["w_gate_up"], full["w_down"])
ys = ep.ep_layer_fwd(so, ep.TorchComm(), full["x"], full["subkeys"], full["W"], om.pack_v(sd, full["V"]), dims.N)
torch.cuda.synchronize()
es = rel_errors(ys.float().cpu().numpy(), y.float().cpu().numpy())
assert es[0] <= 1e-2 and es[1] <= 1e-2, es
y1 = om.layer_fwd(dims, full["x"], full["subkeys"], full["W"], full["V"], full["w_gate_up"], full["w_down"])
torch.cuda.synchronize()
e = rel_errors(y.float().cpu().numpy(), y1.float().cpu().numpy())
print("ERR", e[0], e[1])
dist.destroy_process_group()
'''
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", script], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("ERR")][0]
    e_tok, e_elt = map(float, line.split()[1:])
    assert e_tok <= 1e-2 and e_elt <= 1e-2


def test_bench_multi_two_process_gloo_dry_run():
    """bench.py's N > 1 path launched as the driver does (torchrun, 2 ranks), over gloo
    with host-staged all-to-alls so that both ranks can share this box's one GPU: the
    protocol runs end to end and rank 0 prints one well-formed JSON line."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "2", "--warmup",
           "1", "--config", "C1", "--backend", "gloo", "--no-e2e", "--cpu-seconds", "2"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["scaling"] == "strong" and j["config"]["global_tokens"] == 256
    assert j["parity"]["mismatch"] == 0 and j["parity"]["e_tok"] <= 1e-2 and j["parity"]["e_elt"] <= 1e-2
    assert j["roofline"]["nvlink"]["bytes_per_step_rank0"] > 0 and j["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("vl", [om.V_SLICED])
def test_ep_loopback_c5_per_rank_shape(vl):
    """configs[4] at R = 8 in loopback: N = 2^22 experts (2^19 per virtual rank),
    65,536 tokens (8,192 per rank), K = 512; sampled tokens against the oracle."""
    w = configs.get("C5", v_layout=vl)
    dims, L, R = w.dims, w.L, 8
    full = make_inputs(dims, L, w.seed, skip=("W", "V"))
    ops = ep.LibOps(dims)
    ops.set_mlp(full["w_gate_up"], full["w_down"])
    lpr, n_per = L // R, dims.N // R
    xs = [full["x"][r * lpr:(r + 1) * lpr] for r in range(R)]
    Ws, Vs = [], []
    for r in range(R):
        sh = make_inputs(dims, 1, w.seed, skip=("x", "subkeys", "w_gate_up", "w_down"),
                         expert_rows=(r * n_per, (r + 1) * n_per))
        Ws.append(sh["W"])
        Vs.append(om.pack_v(dims, sh["V"]))
        del sh
    ys = ep.ep_layer_fwd_loopback(ops, xs, full["subkeys"], Ws, Vs, n_per)
    y = torch.cat(ys)
    torch.cuda.synchronize()
    rng = np.random.default_rng(8)
    toks = np.unique(np.concatenate([[0, lpr - 1, lpr, L - 1], rng.choice(L, 60, replace=False)]))
    hr = lambda n, r=None: host_rows(dims, w.seed, n, r)
    x = hr("x", toks)
    sub = hr("subkeys").reshape(1, -1, dims.d)
    lg = oracle.logits(x, sub)
    rt = oracle.route(lg.reshape(len(toks), -1), dims.n_rows, dims.n_cols, dims.top_k)
    used = np.unique(rt["idx"])
    ref = oracle.layer(x, sub, hr("W", used), hr("V", used), dims.n_rows, dims.n_cols, dims.top_k,
                       hr("w_gate_up"), hr("w_down"), id_map=np.stack([used, np.arange(len(used))], 1))
    e_tok, e_elt = rel_errors(y[torch.from_numpy(toks).cuda()].float().cpu().numpy(), ref["y"])
    assert e_tok <= 1e-2 and e_elt <= 1e-2, (e_tok, e_elt)


def test_ep_device_api_one_rank():
    """The fused exchange on the NCCL device API (N3: symmetric windows, peer stores,
    in-kernel LSA barriers) over a real one-rank NCCL communicator -- the only size this
    box has: the layer output equals the host-API expert-parallel path bit for bit (same
    kernels, same message layouts) and the single-GPU layer within 1e-2."""
    script = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2602_05711_b200 import build, distributed as ep, omnimoe as om
from synth.workloads import make_inputs
from tests.helpers import rel_errors
build.build_ep()
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
dims = om.LayerDims(d=256, n_rows=64, n_cols=64, top_k=32, n_heads=2, d_ff=256, v_layout=om.V_SLICED)
full = make_inputs(dims, 384, 7)
Vs = om.pack_v(dims, full["V"])
ops = ep.LibOps(dims); ops.set_mlp(full["w_gate_up"], full["w_down"])
dx = ep.DevExchange(dims, row_cap=384, rec_cap=384 * 64)
y_dev = ep.ep_layer_fwd_dev(ops, dx, full["x"], full["subkeys"], full["W"], Vs, dims.N)
y_host = ep.ep_layer_fwd(ops, ep.TorchComm(), full["x"], full["subkeys"], full["W"], Vs, dims.N)
torch.cuda.synchronize()
print("EQUAL", bool(torch.equal(y_dev, y_host)))
y1 = om.layer_fwd(dims, full["x"], full["subkeys"], full["W"], Vs, full["w_gate_up"], full["w_down"])
torch.cuda.synchronize()
e = rel_errors(y_dev.float().cpu().numpy(), y1.float().cpu().numpy())
print("ERR", e[0], e[1])
dx.close()
dist.destroy_process_group()
'''
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", script], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-3000:])
    assert "EQUAL True" in out.stdout, out.stdout[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("ERR")][0]
    e_tok, e_elt = map(float, line.split()[1:])
    assert e_tok <= 1e-2 and e_elt <= 1e-2
