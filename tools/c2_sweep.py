"""configs[1] router-only sweep: d = 1024, N = 256 x 256, h = 4 heads,
L in {1k, 2k, 4k, 8k, 16k} x K in {1, 4, 16, 64}: omnimoe_route (exact i8 logits + the
selection, key order -- the router API) timed with CUDA events after an L2 flush,
median of 7.  The brute-force index check of every point is
tests/test_gpu_fullsize.py::test_c2_sweep_brute_force.  One JSON line per point."""
import dataclasses
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05711_b200 import build, configs, omnimoe as om  # noqa: E402
from synth.workloads import make_inputs  # noqa: E402

build.build()
w0 = configs.get("C2")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for K in (1, 4, 16, 64):
    for L in (1024, 2048, 4096, 8192, 16384):
        dims = dataclasses.replace(w0.dims, top_k=K)
        inp = make_inputs(dims, L, w0.seed, skip=("W", "V", "w_gate_up", "w_down"))
        ws = om.workspace(dims, L, om.WS_ROUTE)
        ts, lts = [], []
        for it in range(8):
            for what, acc in (("route", ts), ("logits", lts)):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                if what == "route":
                    om.route(dims, inp["x"], inp["subkeys"], ws=ws, want_score=False)
                else:
                    om.router_logits(dims, inp["x"], inp["subkeys"], ws=ws)
                b.record()
                torch.cuda.synchronize()
                if it:
                    acc.append(a.elapsed_time(b))
        ms, lms = statistics.median(ts), statistics.median(lts)
        ops = 2.0 * L * dims.n_heads * (dims.n_rows + dims.n_cols) * dims.d
        print(json.dumps({"config": "C2", "L": L, "K": K, "h": dims.n_heads, "route_ms": ms, "logits_ms": lms,
                          "select_ms": ms - lms, "tokens_per_s": L / (ms / 1e3),
                          "router_gflop": ops / 1e9, "logit_tflops_bf16_equiv": ops / (lms / 1e3) / 1e12}),
              flush=True)
