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
plan = om.schedule(dims, idx.reshape(-1), gate.reshape(-1))
Ws = om.pack_v(dims, inp["W"])
dy = torch.randn(L, dims.d, device="cuda").to(torch.bfloat16)
rd = configs.get(name, group_size=1).dims
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms = []
for i in range(reps + 1):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    om.expert_bwd(rd, inp["x"], inp["W"], inp["V"], Ws, plan, dy)
    b.record()
    torch.cuda.synchronize()
    if i:
        ms.append(a.elapsed_time(b))
t = statistics.median(ms)
M = L * dims.n_heads * dims.top_k
na = int(plan["n_active"].item())
d = dims.d
hbm = na * d * 2 * 2 + na * d * 4 * 2 + L * d * 2 * 2 + L * d * 4 + 16 * M  # W, V once; dW, dV; x, dy; dx; plan
l2 = M * d * 2 * 2 + M * d * 2 + 8 * M * (d // 32)  # x and dy rows per task; W slice per task; pairs per slice
print(json.dumps({"config": name, "ms": t, "tasks": M, "n_active": na, "algorithmic_hbm_bytes": hbm,
                  "hbm_gbs": hbm / t / 1e6, "l2_dataflow_bytes": l2, "l2_gbs": l2 / t / 1e6}))
