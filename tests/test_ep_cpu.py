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
