#!/usr/bin/env python
"""OmniMoE layer-forward benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3a] [--impl ours|reference]

A step is one omnimoe_layer_fwd over one batch of the workload's L tokens (all
of steps a1-a8: route, schedule, expert compute, shared MLP + combine), with
inputs resident in HBM.  Every timed step is preceded by an L2 flush (a 256 MB
write, outside the events); steps are timed with CUDA events on the launching
stream, synchronised and barriered on both sides, max over ranks.
Rank 0 prints one JSON line.  Multi-GPU (torchrun) runs the expert-parallel
layer of paper_2602_05711_b200.distributed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "OmniMoE layer fwd tokens/s + latency ms at 1/2/4/8 B200; HBM GB/s vs peak"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=j.get("hbm_gbs", 6552.0), bf16=j.get("bf16_tflops", 1677.0),
                    bf16_sus=j.get("bf16_tflops_sustained", 1413.9), src="MEASURED_PEAKS.json")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in self.rows:
            if len(r) >= 7:
                for n, v in zip(names, r[3:7]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_a6(dims, L, n_active, M):
    """a6 algorithmic HBM bytes per launch: W and V rows of
    each active expert once (Eq.(vii)) + x read + y_routed write
    (fp32) + plan (token id + gate per task, segment offsets per active expert)."""
    eb = 2 if dims.dtype == 0 else 4
    return (2 * n_active * dims.d * eb + L * dims.d * eb + L * dims.d * 4 + 8 * M + 8 * n_active)


def cpu_oracle_rate(w, n_tokens, nthreads, mode=0):
    """Oracle (as it stands) on a bounded token sample; returns tokens/s, tokens, seconds."""
    import oracle
    from tests.helpers import host_rows
    dims = w.dims
    R = dims.n_rows + dims.n_cols
    sub = host_rows(dims, w.seed, "subkeys", None, mode).reshape(dims.n_heads, R, dims.d)
    wgu = host_rows(dims, w.seed, "w_gate_up", None, mode) if dims.d_ff else None
    wdn = host_rows(dims, w.seed, "w_down", None, mode) if dims.d_ff else None
    chunk = max(1, min(n_tokens, 32))
    total_t, done = 0.0, 0
    for c0 in range(0, n_tokens, chunk):
        toks = np.arange(c0, min(n_tokens, c0 + chunk))
        x = host_rows(dims, w.seed, "x", toks, mode)
        # routing decides which expert rows the oracle needs; regenerate only those (not timed)
        lg = oracle.logits(x, sub, nthreads)
        r = oracle.route(lg.reshape(-1, R), dims.n_rows, dims.n_cols, dims.top_k, oracle.PRODUCT,
                         nthreads=nthreads)
        used = np.unique(r["idx"])
        W = host_rows(dims, w.seed, "W", used, mode)
        V = host_rows(dims, w.seed, "V", used, mode)
        idm = np.stack([used, np.arange(len(used))], 1)
        t0 = time.perf_counter()
        oracle.layer(x, sub, W, V, dims.n_rows, dims.n_cols, dims.top_k, wgu, wdn, id_map=idm,
                     nthreads=nthreads)
        total_t += time.perf_counter() - t0
        done += len(toks)
    return done / total_t, done, total_t


def rank_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lr


def run_reference(args):
    """--impl reference: the oracle (CPU, host cores) on bounded samples of the same workload."""
    ws, rk, _ = rank_info()
    if rk != 0:
        return 0
    from paper_2602_05711_b200 import configs
    w = configs.get(args.config)
    nth = os.cpu_count() or 1
    n_tok = args.ref_tokens
    for _ in range(args.warmup if args.warmup <= 1 else 1):
        cpu_oracle_rate(w, min(n_tok, 8), nth)
    times = []
    for _ in range(args.steps):
        rate, done, t = cpu_oracle_rate(w, n_tok, nth)
        times.append(t)
    rate = args.steps * n_tok / sum(times)
    ms = 1000.0 * w.L / rate
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "d": w.dims.d, "n_rows": w.dims.n_rows, "n_cols": w.dims.n_cols,
                       "top_k": w.dims.top_k, "n_heads": w.dims.n_heads, "d_ff": w.dims.d_ff, "tokens": w.L},
            "cpu_baseline": {"value": rate, "unit": "tokens/s", "cores": nth, "kind": "oracle",
                             "sample": f"{n_tok} tokens of {w.name} per step (oracle layer: fp64 canonical "
                                       f"logits, product top-K, token-centric routed branch, shared MLP); "
                                       f"ms_per_step extrapolates to the full {w.L}-token batch"},
            "e2e": {"value": rate, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3a")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-tokens", type=int, default=64)
    ap.add_argument("--ref-tokens", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    ws, rk, lr = rank_info()
    torch.cuda.set_device(lr)
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", lr))
    from paper_2602_05711_b200 import build, configs, omnimoe as om
    build.build()
    from synth.workloads import make_inputs
    w = configs.get(args.config)
    dims = w.dims
    L = w.L
    if ws > 1:
        from paper_2602_05711_b200 import distributed as ep
        return ep.bench_main(args, w, ws, rk, lr)

    inp = make_inputs(dims, L, w.seed)
    lws = om.workspace(dims, L, om.WS_LAYER)
    y = torch.empty((L, dims.d), dtype=dims.torch_dtype, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()

    def step():
        om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"),
                     inp.get("w_down"), y=y, ws=lws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = om.last_launch_count()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(lr) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(st)
            step()
            ev[i][1].record(st)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.mean(step_ms)

    # ---- per-stage breakdown through the individual C-ABI calls (same inputs) ----
    idx = torch.empty((L, dims.n_heads, dims.top_k), dtype=torch.int32, device="cuda")
    rws = om.workspace(dims, L, om.WS_ROUTE)
    M = L * dims.n_heads * dims.top_k
    plan = om.new_plan(dims.N, M, "cuda")
    sws = om.workspace(dims, M, om.WS_SCHEDULE)
    yr = torch.empty((L, dims.d), dtype=torch.float32, device="cuda")
    stages = {"route": [], "schedule": [], "expert": [], "shared_mlp": []}
    for i in range(max(3, args.steps // 2)):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
        flush.zero_()
        e[0].record(st)
        idx, gate, _ = om.route(dims, inp["x"], inp["subkeys"], ws=rws, want_score=False)
        e[1].record(st)
        om.schedule(dims, idx.reshape(-1), gate.reshape(-1), plan=plan, ws=sws)
        e[2].record(st)
        yr.zero_()
        flush.zero_()
        e[3].record(st)
        om.expert_fwd(dims, inp["x"], inp["W"], inp["V"], plan, y_routed=yr, accumulate=True)
        e[4].record(st)
        if dims.d_ff:
            om.shared_mlp(dims, inp["x"], inp["w_gate_up"], inp["w_down"], y_routed=yr, y=y)
        e[5].record(st)
        torch.cuda.synchronize()
        if i == 0:
            continue  # first pass allocates workspaces
        stages["route"].append(e[0].elapsed_time(e[1]))
        stages["schedule"].append(e[1].elapsed_time(e[2]))
        stages["expert"].append(e[3].elapsed_time(e[4]))
        stages["shared_mlp"].append(e[4].elapsed_time(e[5]))
    stage_ms = {k: statistics.mean(v) for k, v in stages.items()}
    n_active = int(plan["n_active"].item())

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        xh = inp["x"].cpu().pin_memory()
        yh = torch.empty(y.shape, dtype=y.dtype).pin_memory()
        xd = torch.empty_like(inp["x"])
        for _ in range(2):
            xd.copy_(xh, non_blocking=True)
            om.layer_fwd(dims, xd, inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"), inp.get("w_down"), y=y, ws=lws)
            yh.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(args.steps):
            flush.zero_()
            a.record(st)
            xd.copy_(xh, non_blocking=True)
            om.layer_fwd(dims, xd, inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"), inp.get("w_down"), y=y, ws=lws)
            yh.copy_(y, non_blocking=True)
            b.record(st)
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        e2e_ms = tot / args.steps
        eb = 2 if dims.dtype == 0 else 4
        e2e = {"value": L / (e2e_ms / 1000.0), "unit": "tokens/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": L * dims.d * eb, "d2h_bytes_per_step": L * dims.d * eb}

    pk = peaks()
    a6_bytes = algorithmic_a6(dims, L, n_active, M)
    a6_gbs = a6_bytes / (stage_ms["expert"] / 1000.0) / 1e9
    roofline = {"kernel": "expert_warp_kernel (a6)", "bound": "hbm", "achieved": a6_gbs, "peak": pk["hbm"],
                "unit": "GB/s", "frac": a6_gbs / pk["hbm"], "traffic": None,
                "algorithmic_bytes_per_launch": a6_bytes, "avg_launch_ms": stage_ms["expert"],
                "peak_source": pk["src"] + " hbm_gbs (copy)"}
    # other kernels' rooflines (context)
    R = dims.n_rows + dims.n_cols
    router_flops = 2.0 * L * dims.n_heads * R * dims.d
    mlp_flops = 6.0 * L * dims.d * dims.d_ff

    cpu = None
    if not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        rate, done, t = cpu_oracle_rate(w, args.cpu_tokens, nth)
        cpu = {"value": rate, "unit": "tokens/s", "cores": nth, "kind": "oracle",
               "sample": f"{done} tokens of {w.name} (oracle layer: fp64 canonical logits, product top-K, "
                         f"token-centric routed branch, shared MLP), {t:.1f} s on {nth} threads"}

    line = {
        "metric": METRIC, "value": L / (ms / 1000.0), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "latency_ms": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": w.name, "d": dims.d, "n_rows": dims.n_rows, "n_cols": dims.n_cols,
                   "top_k": dims.top_k, "n_heads": dims.n_heads, "d_ff": dims.d_ff, "tokens": L,
                   "router": "exact (int8 tcgen05 limbs)", "parallelism": "single-gpu",
                   "l2": "flushed (256 MB write) before every timed step"},
        "stage_ms": stage_ms, "n_active": n_active, "tasks": M,
        "step_ms_min_max": [min(step_ms), max(step_ms)],
        "roofline": roofline,
        "other_rooflines": {
            "router_gemm_a1": {"tflop": router_flops / 1e12},
            "shared_mlp_a7": {"tflop": mlp_flops / 1e12,
                              "achieved_tflops": mlp_flops / (stage_ms["shared_mlp"] / 1e3) / 1e12 if dims.d_ff else None,
                              "peak": pk["bf16_sus"]}},
        "e2e": e2e, "cpu_baseline": cpu,
        "gpu_launches": launches * args.steps, "launches_per_step": launches,
        "clocks": clk.summary(),
        "context": "paper: 6.7 ms OmniMoE vs 73 ms PEER at 4,096 tokens on A100 (PAPER:368), different shape",
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
