"""Expert-parallel exchange protocol on CPU (-m "not gpu"): two gloo ranks run
paper_2602_05711_b200.distributed.ep_layer_fwd with oracle-backed kernels
(tests/ep_ref.py) on half of the tokens and half of the expert rows each; the
result must equal the single-process oracle layer (Eq.MoE) on all tokens."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

D, NR, NC, K, H, L, DFF = 16, 8, 8, 5, 2, 24, 8


def _inputs():
    ex = synth.default_exponents(D, DFF)
    dec = lambda tid, shape: torch.from_numpy(
        synth.bf16_bits_to_f64(synth.gen_bf16_bits(4, tid, shape, ex[tid])))
    return dict(x=dec(synth.TID_X, (L, D)), sub=dec(synth.TID_SUBKEYS, (H, NR + NC, D)),
                W=dec(synth.TID_W, (NR * NC, D)), V=dec(synth.TID_V, (NR * NC, D)),
                wgu=dec(synth.TID_W_GATE_UP, (2 * DFF, D)), wdn=dec(synth.TID_W_DOWN, (D, DFF)))


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_05711_b200 import distributed as ep
    from tests.ep_ref import RefOps
    inp = _inputs()
    n_per = NR * NC // world
    lpr = L // world
    ops = RefOps(NR, NC, K, inp["wgu"], inp["wdn"])
    y = ep.ep_layer_fwd(ops, ep.TorchComm(), inp["x"][rank * lpr:(rank + 1) * lpr].contiguous(), inp["sub"],
                        ep.shard_rows(inp["W"], world, rank), ep.shard_rows(inp["V"], world, rank), n_per)
    torch.save(y, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_ep_gloo_matches_single_process_oracle(world, tmp_path):
    out = str(tmp_path / "y")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, start_method="spawn")
    y = torch.cat([torch.load(f"{out}.{r}") for r in range(world)]).numpy()
    inp = _inputs()
    ref = oracle.layer(inp["x"].numpy(), inp["sub"].numpy(), inp["W"].numpy(), inp["V"].numpy(), NR, NC, K,
                       inp["wgu"].numpy(), inp["wdn"].numpy())
    np.testing.assert_allclose(y, ref["y"], rtol=1e-12, atol=1e-12)


def test_ep_loopback_reference_ops_match_oracle():
    """The in-process loopback driver (what the single-GPU EP test uses) with the
    same reference kernels, R = 4 virtual ranks."""
    from paper_2602_05711_b200 import distributed as ep
    from tests.ep_ref import RefOps
    inp = _inputs()
    R = 4
    ops = RefOps(NR, NC, K, inp["wgu"], inp["wdn"])
    lpr = L // R
    ys = ep.ep_layer_fwd_loopback(ops, [inp["x"][r * lpr:(r + 1) * lpr] for r in range(R)], inp["sub"],
                                  [ep.shard_rows(inp["W"], R, r) for r in range(R)],
                                  [ep.shard_rows(inp["V"], R, r) for r in range(R)], NR * NC // R)
    ref = oracle.layer(inp["x"].numpy(), inp["sub"].numpy(), inp["W"].numpy(), inp["V"].numpy(), NR, NC, K,
                       inp["wgu"].numpy(), inp["wdn"].numpy())
    np.testing.assert_allclose(torch.cat(ys).numpy(), ref["y"], rtol=1e-12, atol=1e-12)


def _skewed_routing(world):
    """Uneven fan-out: tasks concentrated on shard 0, some tokens reaching one shard
    only, shard world-1 receiving nothing from the last rank's tokens."""
    rng = np.random.default_rng(11)
    N, hk = NR * NC, H * K
    n_per = N // world
    idx = np.empty((L, hk), np.int64)
    lpr = L // world
    for l in range(L):
        r = l // lpr
        if l % 3 == 0:      # one destination only (shard 0)
            pool = np.arange(0, n_per)
        elif r == world - 1:  # the last rank's tokens never reach the last shard
            pool = np.arange(0, (world - 1) * n_per)
        else:
            pool = np.arange(N)
        idx[l] = rng.choice(pool, hk, replace=False)
    gate = rng.random((L, hk))
    return idx, gate / gate.sum(1, keepdims=True)


class _SkewOps:
    """RefOps with the routing replaced by a fixed skewed assignment (global token ids
    recovered from the row offset of the rank's slice)."""

    def __init__(self, base, idx, gate, l0):
        self.base, self.idx, self.gate, self.l0 = base, idx, gate, l0

    def route(self, x, subkeys):
        n = x.shape[0]
        return (torch.from_numpy(self.idx[self.l0:self.l0 + n]), torch.from_numpy(self.gate[self.l0:self.l0 + n]))

    def __getattr__(self, k):
        return getattr(self.base, k)


def _worker_skew(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_05711_b200 import distributed as ep
    from tests.ep_ref import RefOps
    inp = _inputs()
    idx, gate = _skewed_routing(world)
    lpr = L // world
    ops = _SkewOps(RefOps(NR, NC, K, inp["wgu"], inp["wdn"]), idx, gate, rank * lpr)
    y = ep.ep_layer_fwd(ops, ep.TorchComm(), inp["x"][rank * lpr:(rank + 1) * lpr].contiguous(), inp["sub"],
                        ep.shard_rows(inp["W"], world, rank), ep.shard_rows(inp["V"], world, rank),
                        NR * NC // world)
    torch.save(y, f"{out_path}.{rank}")
    dist.barrier()
    dist.destroy_process_group()


def test_ep_gloo_four_ranks_uneven_fanout(tmp_path):
    """World size 4, skewed routing (empty (source, destination) blocks, one-destination
    tokens): the exchange still reproduces the single-process composition exactly."""
    world = 4
    out = str(tmp_path / "y")
    mp.start_processes(_worker_skew, args=(world, _free_port(), out), nprocs=world, start_method="spawn")
    y = torch.cat([torch.load(f"{out}.{r}") for r in range(world)]).numpy()
    inp = _inputs()
    idx, gate = _skewed_routing(world)
    dest = idx // (NR * NC // world)
    assert (dest[(L // world) * (world - 1):] != world - 1).all() and (dest[::3] == 0).all()
    ref = oracle.routed_token_centric(inp["x"].numpy(), inp["W"].numpy(), inp["V"].numpy(), idx.astype(np.int32),
                                      gate) + oracle.shared_mlp(inp["x"].numpy(), inp["wgu"].numpy(),
                                                                inp["wdn"].numpy())
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
