"""Per-kernel durations of omnimoe_layer_fwd under normal (unserialised) execution, via
torch.profiler (CUPTI): python tools/layer_prof.py C5 [rows|sliced] [reps]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_05711_b200 import configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3a"
layout = om.V_ROWS if (len(sys.argv) > 2 and sys.argv[2] == "rows") else om.V_SLICED
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = configs.get(name, v_layout=layout)
inp = make_inputs(w.dims, w.L, w.seed)
if layout == om.V_SLICED:
    inp["V"] = om.pack_v(w.dims, inp["V"])
ws = om.workspace(w.dims, w.L, om.WS_LAYER)
y = torch.empty((w.L, w.dims.d), dtype=w.dims.torch_dtype, device="cuda")
run = lambda: om.layer_fwd(w.dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"),
                           inp.get("w_down"), y=y, ws=ws)
run()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(reps):
    run()
ev[1].record()
torch.cuda.synchronize()
print(f"layer {name}: {ev[0].elapsed_time(ev[1]) / reps:.3f} ms (warm, no flush)")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
tot = collections.OrderedDict()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:50]
        tot[k] = tot.get(k, 0.0) + e.device_time / 1000.0 / reps
s = 0.0
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    s += v
    print(f"{v:9.3f} ms  {k}")
print(f"{s:9.3f} ms  total kernel time per layer")
