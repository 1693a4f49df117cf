"""Per-kernel durations of omnimoe_expert_bwd (torch.profiler / CUPTI): python tools/bwd_prof.py C3a"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_05711_b200 import configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3a"
w = configs.get(name, v_layout=om.V_SLICED, route_order=om.ORDER_CANDIDATE)
dims, L = w.dims, w.L
inp = make_inputs(dims, L, w.seed)
idx, gate, _ = om.route(dims, inp["x"], inp["subkeys"], want_score=False)
rd = om.bwd_dims(dims)
plan = om.schedule(rd, idx.reshape(-1), gate.reshape(-1))
Ws = om.pack_v(dims, inp["W"])
dy = torch.randn(L, dims.d, device="cuda").to(torch.bfloat16)
run = lambda: om.expert_bwd(rd, inp["x"], inp["W"], inp["V"], Ws, plan, dy)
run()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        run()
    torch.cuda.synchronize()
tot = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name[:60]] += e.device_time_total / 1000.0 / 3
for k, v in tot.most_common(12):
    print(f"{v:9.3f} ms  {k}")
