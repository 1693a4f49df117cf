"""Measure |fast tcgen05 logit - canonical fp64 logit| per config (DESIGN.md
"Certified routing": cert_eps = 8 x the max observed error, >= 1e7 logits)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05711_b200 import build, configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

build.build()
out = {}
for name in sys.argv[1:] or ["C1", "C2", "C3a", "C4", "C5"]:
    w = configs.get(name)
    R = w.dims.n_rows + w.dims.n_cols
    L = max(256, min(w.L, (10_000_000 // (R * w.dims.n_heads)) + 1))
    worst, worst_rel, n = 0.0, 0.0, 0
    for seed in (w.seed, w.seed + 10):
        inp = make_inputs(w.dims, L, seed, skip=("W", "V", "w_gate_up", "w_down"))
        f = om.router_logits(w.dims, inp["x"], inp["subkeys"], canonical=False)
        c = om.router_logits(w.dims, inp["x"], inp["subkeys"], canonical=True)
        torch.cuda.synchronize()
        d = (f.double() - c.double()).abs()
        worst = max(worst, d.max().item())
        worst_rel = max(worst_rel, (d / c.double().abs().clamp_min(1e-3)).max().item())
        n += c.numel()
    out[name] = {"logits": n, "max_abs_err": worst, "max_rel_err": worst_rel, "eps_8x": 8 * worst,
                 "d": w.dims.d, "L_sampled": L}
    print(name, out[name], flush=True)
print(json.dumps(out))
