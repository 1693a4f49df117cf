"""N2 measurement: routed-branch backward (omnimoe_expert_bwd) on a workload's routing.
    python tools/bwd_bench.py [C3a] [reps]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_05711_b200 import configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = configs.get(name, v_layout=om.V_SLICED, route_order=om.ORDER_CANDIDATE)
dims, L = w.dims, w.L
inp = make_inputs(dims, L, w.seed)
idx, gate, _ = om.route(dims, inp["x"], inp["subkeys"], want_score=False)
rd = om.bwd_dims(dims)  # group size 1, one V band (the backward's plan)
plan = om.schedule(rd, idx.reshape(-1), gate.reshape(-1))
Ws = om.pack_v(dims, inp["W"])
dy = torch.randn(L, dims.d, device="cuda").to(torch.bfloat16)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms, parts = [], {"expert_bwd": [], "router_bwd": [], "mlp_bwd": []}
for i in range(reps + 1):
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    dx, dW, dV, dg = om.expert_bwd(rd, inp["x"], inp["W"], inp["V"], Ws, plan, dy)
    ev[1].record()
    om.router_bwd(dims, inp["x"], inp["subkeys"], idx, gate, dg.reshape(gate.shape), dx=dx, accumulate_dx=True)
    ev[2].record()
    if dims.d_ff:
        om.shared_mlp_bwd(dims, inp["x"], inp["w_gate_up"], inp["w_down"], dy, dx=dx, accumulate_dx=True)
    ev[3].record()
    torch.cuda.synchronize()
    if i:
        ms.append(ev[0].elapsed_time(ev[1]))
        for k, (u, v) in zip(parts, [(0, 1), (1, 2), (2, 3)]):
            parts[k].append(ev[u].elapsed_time(ev[v]))
t = statistics.median(ms)
part_ms = {k: statistics.median(v) for k, v in parts.items()}
M = L * dims.n_heads * dims.top_k
na = int(plan["n_active"].item())
d = dims.d
hbm = na * d * 2 * 2 + na * d * 4 * 2 + L * d * 2 * 2 + L * d * 4 + 16 * M  # W, V once; dW, dV; x, dy; dx; plan
l2 = M * d * 2 * 2 + M * d * 2 + 8 * M * (d // 64)  # x and dy rows per task; W slice per task; pairs per slice
print(json.dumps({"config": name, "layer_bwd_ms": sum(part_ms.values()), "part_ms": part_ms, "ms": t, "tasks": M, "n_active": na, "algorithmic_hbm_bytes": hbm,
                  "hbm_gbs": hbm / t / 1e6, "l2_dataflow_bytes": l2, "l2_gbs": l2 / t / 1e6}))
