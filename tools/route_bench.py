"""Times omnimoe_route and its a1 part (exact logits) per config; select = route - logits."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05711_b200 import build, configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

build.build()
out = {}
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3a", "C3b", "C4", "C5"]):
    w = configs.get(name)
    L = min(w.L, 16384)
    inp = make_inputs(w.dims, L, w.seed, skip=("W", "V", "w_gate_up", "w_down"))
    ws = om.workspace(w.dims, L, om.WS_ROUTE)
    res = {}
    lws = om.workspace(w.dims, L, om.WS_LAYER) if False else None
    for what in ("logits", "route"):
        ts = []
        for it in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if what == "logits":
                om.router_logits(w.dims, inp["x"], inp["subkeys"], ws=ws)
            else:
                om.route(w.dims, inp["x"], inp["subkeys"], ws=ws, want_score=False)
            b.record()
            torch.cuda.synchronize()
            if it:
                ts.append(a.elapsed_time(b))
        res[what] = sorted(ts)[len(ts) // 2]
    res["select"] = res["route"] - res["logits"]
    res["tokens"] = L
    out[name] = res
    print(name, res, flush=True)
print(json.dumps(out))
