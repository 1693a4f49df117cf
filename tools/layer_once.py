"""Run omnimoe_layer_fwd a few times on a workload (for ncu captures).
    python tools/layer_once.py C3a [rows|sliced] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_05711_b200 import configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3a"
layout = om.V_ROWS if (len(sys.argv) > 2 and sys.argv[2] == "rows") else om.V_SLICED
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
over = {k: int(v) for k, v in (a.split("=") for a in sys.argv[4:])}
w = configs.get(name, v_layout=layout, **over)
inp = make_inputs(w.dims, w.L, w.seed)
if layout == om.V_SLICED:
    inp["V"] = om.pack_v(w.dims, inp["V"])
ws = om.workspace(w.dims, w.L, om.WS_LAYER)
y = torch.empty((w.L, w.dims.d), dtype=w.dims.torch_dtype, device="cuda")
for _ in range(reps):
    om.layer_fwd(w.dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"), inp.get("w_down"),
                 y=y, ws=ws)
torch.cuda.synchronize()
print("ok", name, layout)
