"""Times schedule + expert_fwd (a4-a6) for several group sizes B on one workload."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05711_b200 import build, configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

build.build()
name = sys.argv[1] if len(sys.argv) > 1 else "C3a"
# entries "B" or "B:Tb" (group size, token blocks; Tb 0 = library choice)
specs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "1024", "4096"]
Bs = [tuple(int(v) for v in (s + ":0").split(":")[:2]) for s in specs]
w = configs.get(name)
inp = make_inputs(w.dims, w.L, w.seed, skip=("w_gate_up", "w_down"))
idx, gate, _ = om.route(w.dims, inp["x"], inp["subkeys"], want_score=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {}
for B, Tb in Bs:
    dims = configs.get(name, group_size=B, token_blocks=Tb).dims
    M = idx.numel()
    plan = om.new_plan(dims.N, M, "cuda")
    sws = om.workspace(dims, M, om.WS_SCHEDULE)
    ews = om.workspace(dims, w.L, om.WS_EXPERT)
    y = torch.empty((w.L, dims.d), dtype=torch.float32, device="cuda")
    ts, te = [], []
    for it in range(6):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        flush.zero_()
        e[0].record()
        om.schedule(dims, idx.reshape(-1), gate.reshape(-1), plan=plan, ws=sws)
        e[1].record()
        flush.zero_()
        e[2].record()
        om.expert_fwd(dims, inp["x"], inp["W"], inp["V"], plan, y_routed=y, ws=ews)
        e[3].record()
        torch.cuda.synchronize()
        if it:
            ts.append(e[0].elapsed_time(e[1]))
            te.append(e[2].elapsed_time(e[3]))
    key = f"{B}:{om.token_blocks(dims, w.L)}"
    out[key] = {"schedule_ms": sorted(ts)[len(ts) // 2], "expert_ms": sorted(te)[len(te) // 2],
              "n_runs": int(plan["n_runs"].item()) if B > 1 else None}
    print(name, key, out[key], flush=True)
print(json.dumps({name: out}))
