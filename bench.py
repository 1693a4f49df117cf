#!/usr/bin/env python
"""OmniMoE layer-forward benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3a] [--impl ours|reference]

A step is one OmniMoE layer forward (steps a1-a8 of DESIGN.md: route, schedule,
grouped expert compute, shared MLP + combine) over one batch of the workload's
L tokens per GPU, inputs resident in HBM.  Every timed step is preceded by an L2
flush (a 256 MB write, outside the events); steps are timed with CUDA events on
the launching stream, barrier + synchronize on both sides, max over ranks.

N = 1: omnimoe_layer_fwd (the single-GPU C-ABI call).  N > 1 (torchrun): the
expert-parallel layer of paper_2602_05711_b200.distributed -- each rank keeps L
tokens (weak scaling) and 1/N of the expert table's rows; NCCL all-to-all
dispatch and combine.  Rank 0 prints ONE JSON line.

--impl reference: the CPU oracle (oracle/, as it stands) on a bounded token
sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import dataclasses
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
                    bf16_sus=j.get("bf16_tflops_sustained", 1413.9), src="measured (MEASURED_PEAKS.json)")
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
            time.sleep(0.3)
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
        ok = [r for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        sm = [float(r[0]) for r in ok]
        mx = [float(r[1]) for r in ok if r[1].replace(".", "").isdigit()]
        reasons = sorted({n for r in ok for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def rank_info():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def expected_eta(dims, L):
    """Tasks per active expert under uniform routing: M / (N (1 - (1 - 1/N)^M))."""
    import math
    N, M = dims.N, L * dims.n_heads * dims.top_k
    return M / (N * -math.expm1(-M / N))


# measured L2 -> SM gather ceilings of this B200 (tools/l2_ceiling.cu, profiles/r2/l2_ceiling/):
# random pieces from a 64 MB L2-resident table with 256-bit loads
L2_GATHER_GBS = {"piece128": 18757.0, "row4k": 19414.0}


def a6_algorithmic_bytes(dims, L, n_active, M):
    """a6 algorithmic HBM bytes per launch: W and V rows of every
    active expert once (D_expert) + x read + y_routed fp32 write +
    plan (token + gate per task, offsets per active expert)."""
    eb = 2 if dims.dtype == 0 else 4
    return 2 * n_active * dims.d * eb + L * dims.d * eb + L * dims.d * 4 + 8 * M + 8 * n_active


def ncu_traffic(config, kernel):
    """dram bytes per launch of `kernel` from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "r2", "ncu_summary.json")
    if not os.path.exists(p):
        return None, None
    j = json.load(open(p))
    rec = j.get(config, {}).get(kernel)
    if not rec:
        return None, None
    return rec.get("dram_bytes"), rec.get("source")


# ---------------------------------------------------------------- CPU oracle
def cpu_oracle_rate(w, target_s, max_tokens, nthreads, inp=None, gpu=None):  # noqa: C901
    """The oracle layer (as it stands) on a bounded token sample.  Expert rows are
    taken from the seeded generator (the device twin's tables when ``inp`` holds
    them -- bit-identical to the host generator, tests/test_gpu_parity.py -- else
    the host twins); only the oracle call is timed.  The sample grows in
    chunks of 32 tokens until ~target_s seconds of oracle time.

    gpu = (y, idx) of the timed layer (host arrays): the same sample then yields
    the north star's parity counters -- token-heads whose id set differs from the
    oracle's (mismatch), of those the ones inside the 1e-6 score-gap allowance
    (allowed, reading Q10) and the rest (disallowed) -- and e_tok / e_elt (Q17)."""
    import oracle
    from tests.helpers import host_rows, rel_errors, routing_counts
    dims = w.dims
    R = dims.n_rows + dims.n_cols
    sub = host_rows(dims, w.seed, "subkeys").reshape(dims.n_heads, R, dims.d)
    wgu = host_rows(dims, w.seed, "w_gate_up") if dims.d_ff else None
    wdn = host_rows(dims, w.seed, "w_down") if dims.d_ff else None

    def rows(name, used):
        if inp is not None and name in inp:
            return inp[name][torch.from_numpy(used).to(inp[name].device)].double().cpu().numpy()
        return host_rows(dims, w.seed, name, used)

    total_t, done, chunk = 0.0, 0, 32
    par = {"tokens": 0, "token_heads": 0, "mismatch": 0, "allowed": 0, "disallowed": 0, "gate_err": 0.0,
           "e_tok": 0.0, "e_elt": 0.0}
    while done < max_tokens and total_t < target_s:
        toks = np.arange(done, min(max_tokens, done + chunk)) % w.L
        x = host_rows(dims, w.seed, "x", toks)
        lg = oracle.logits(x, sub, nthreads)   # routing decides which rows the oracle needs (not timed)
        r = oracle.route(lg.reshape(-1, R), dims.n_rows, dims.n_cols, dims.top_k, oracle.PRODUCT, nthreads=nthreads)
        used = np.unique(r["idx"])
        W, V = rows("W", used), rows("V", used)
        idm = np.stack([used, np.arange(len(used))], 1)
        t0 = time.perf_counter()
        ref = oracle.layer(x, sub, W, V, dims.n_rows, dims.n_cols, dims.top_k, wgu, wdn, id_map=idm,
                           nthreads=nthreads)
        total_t += time.perf_counter() - t0
        done += len(toks)
        if gpu is not None:
            gy, gidx, ggate = gpu
            K = dims.top_k
            c = routing_counts(gidx[toks].reshape(-1, K), ggate[toks].reshape(-1, K), r, lg.reshape(-1, R),
                               dims.n_rows, dims.n_cols)
            et, ee = rel_errors(gy[toks], ref["y"])
            par["tokens"] += len(toks)
            for k in ("token_heads", "mismatch", "allowed", "disallowed"):
                par[k] += c[k]
            par["e_tok"], par["e_elt"] = max(par["e_tok"], et), max(par["e_elt"], ee)
            par["gate_err"] = max(par["gate_err"], c["gate_err"])
    return done / total_t, done, total_t, par


def run_reference(args, w):
    """--impl reference: the oracle on the host cores, bounded sample per step, on the
    workload the other arm times (same config dict)."""
    ws, rk, _ = rank_info()
    if rk != 0:
        return 0
    nth = os.cpu_count() or 1
    per_step_s = max(2.0, args.ref_seconds / max(args.steps, 1))
    tables = None  # expert rows from the generator's host twin: nothing of this arm runs on the GPU
    cpu_oracle_rate(w, 0.5, 32, nth, tables)  # warm-up (page-in, thread pool)
    rates, toks = [], 0
    for _ in range(args.steps):
        rate, done, _t, _ = cpu_oracle_rate(w, per_step_s, 1 << 20, nth, tables)
        rates.append(rate)
        toks += done
    rate = statistics.mean(rates)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * w.L / rate,
            "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _arm_config(w, args, ws),
            "timing_note": ("each step times a bounded token sample of the batch on the host cores; value = "
                            "sampled tokens / oracle seconds, ms_per_step extrapolates it to the whole batch"),
            "cpu_baseline": {"value": rate, "unit": "tokens/s", "cores": nth, "kind": "oracle",
                             "sample": f"{toks} tokens of {w.name} over {args.steps} steps (~{per_step_s:.0f} s of "
                                       f"oracle time each): exact logits, product top-K, token-centric routed "
                                       f"branch, shared MLP; ms_per_step extrapolates to the {w.L}-token batch"},
            "e2e": {"value": rate, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _arm_config(w, args, ws):
    """The config dict both arms print (the driver compares them): the workload, and for one
    GPU the executor the layer runs, for N > 1 the expert-parallel layout."""
    from paper_2602_05711_b200 import omnimoe as om
    dims = w.dims
    if ws > 1:
        return dict(_config_dict(w, f"ep{ws} (experts row-sharded, tokens data-parallel, {args.backend} all-to-all)"),
                    global_tokens=w.L, tokens_per_gpu=w.L // ws, backend=args.backend, exchange=args.exchange)
    return dict(_config_dict(w, "single-gpu"), group_size=om.group_size(dims), expert_kernel=args.expert_kernel,
                v_layout="sliced" if dims.v_layout == om.V_SLICED else "rows",
                executor={om.EXPERT_TOKEN: "token-centric (eta < 2: no expert reuse; ECS skipped)",
                          om.EXPERT_DENSE: "dense tcgen05 GEMMs (K >= N/40; ECS skipped)",
                          om.EXPERT_SLICED: "SLICED (ECS pass Z + slice-major pass V)",
                          om.EXPERT_GROUP: "grouped ECS (rows)",
                          om.EXPERT_WARP: "expert-major ECS (rows)"}[om.layer_executor(dims, w.L)],
                eta=expected_eta(dims, w.L))


def _config_dict(w, parallelism):
    d = w.dims
    return {"workload": w.name, "d": d.d, "n_rows": d.n_rows, "n_cols": d.n_cols, "N": d.N, "top_k": d.top_k,
            "n_heads": d.n_heads, "d_ff": d.d_ff, "tokens_per_gpu": w.L, "parallelism": parallelism,
            "router": "exact (RN32 of the exact dot product; tcgen05 kind::i8 limbs)",
            "l2": "flushed (256 MB write) before every timed step"}


# ---------------------------------------------------------------- N = 1
def bench_single(args, w, lr):
    from paper_2602_05711_b200 import omnimoe as om
    from synth.workloads import make_inputs
    dims, L = w.dims, w.L
    inp = make_inputs(dims, L, w.seed)
    oinp = dict(inp)  # the oracle sample reads expert rows in the [N][d] layout
    if dims.v_layout == om.V_SLICED:  # one-time weight re-layout (not part of a step)
        inp["V"] = om.pack_v(dims, inp["V"])
        torch.cuda.synchronize()
    lws = om.workspace(dims, L, om.WS_LAYER)
    y = torch.empty((L, dims.d), dtype=dims.torch_dtype, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()

    def step(x=None):
        om.layer_fwd(dims, inp["x"] if x is None else x, inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"),
                     inp.get("w_down"), y=y, ws=lws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = om.LAUNCHES
    with ClockSampler(lr) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(st)
            step()
            ev[i][1].record(st)
        torch.cuda.synchronize()
    launches = om.LAUNCHES - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = statistics.mean(step_ms)

    ablation = []
    if dims.expert_kernel == om.EXPERT_TOKEN:
        ablation.append("w/o Expert-Centric Scheduling (token-centric executor, PAPER:396)")
    if dims.router == om.ROUTER_DENSE:
        ablation.append("w/o Cartesian Product Router (dense gate projection, PAPER:395, 414)")
    if args.no_shared_mlp:
        ablation.append("w/o Shared Dense MLP (PAPER:394)")
    if ablation:  # ablation run (PAPER Table 4 rows): the layer time is the result
        print(json.dumps({"metric": METRIC, "value": L / (ms / 1000.0), "unit": "tokens/s", "n_gpus": 1,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                          "data": "synthetic", "config": dict(_config_dict(w, "single-gpu"), ablation=ablation),
                          "workspace_bytes": lws.numel(), "gpu_launches": launches, "clocks": clk.summary()}),
              flush=True)
        return 0
    # ---- per-stage breakdown through the individual C-ABI calls (same inputs) ----
    M = L * dims.n_heads * dims.top_k
    rdims = dataclasses.replace(dims, route_order=om.ORDER_CANDIDATE)  # the layer's routing (no final sort)
    rws = om.workspace(rdims, L, om.WS_ROUTE)
    plan = om.new_plan(dims.N, M, "cuda", dims=dims)
    sws = om.workspace(dims, M, om.WS_SCHEDULE)
    ews = om.workspace(dims, L, om.WS_EXPERT)
    yr = torch.empty((L, dims.d), dtype=torch.float32, device="cuda")
    stages = {"route_a1_a3": [], "schedule_a4_a5": [], "expert_a6": [], "shared_mlp_a7_a8": []}
    sliced = dims.v_layout == om.V_SLICED
    token = om.layer_executor(dims, L) == om.EXPERT_TOKEN  # low eta: the layer skips ECS
    dense = om.layer_executor(dims, L) == om.EXPERT_DENSE  # high eta: two GEMMs
    dws = om.workspace(dims, L, om.WS_LAYER) if dense else None  # (covers the dense scratch)
    passes = {"a6_pass_z": [], "a6_pass_v": []}
    for i in range(max(4, args.steps)):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        flush.zero_()
        e[0].record(st)
        idx, gate, _ = om.route(rdims, inp["x"], inp["subkeys"], ws=rws, want_score=False)
        e[1].record(st)
        om.schedule(dims, idx.reshape(-1), gate.reshape(-1), plan=plan, ws=sws)
        e[2].record(st)
        yr.zero_()
        flush.zero_()
        e[3].record(st)
        if token:
            om.expert_fwd_tokens(dims, inp["x"], inp["W"], inp["V"], idx, gate, y_routed=yr, accumulate=True)
        elif dense:
            om.expert_fwd_dense(dims, inp["x"], inp["W"], inp["V"], idx, gate, y_routed=yr, ws=dws)
        elif sliced:  # the two passes of the SLICED executor, timed apart
            om.expert_fwd(dims, inp["x"], inp["W"], inp["V"], plan, y_routed=yr, accumulate=True, ws=ews, passes=1)
            e[6].record(st)
            om.expert_fwd(dims, inp["x"], inp["W"], inp["V"], plan, y_routed=yr, accumulate=True, ws=ews, passes=2)
        else:
            om.expert_fwd(dims, inp["x"], inp["W"], inp["V"], plan, y_routed=yr, accumulate=True, ws=ews)
        e[4].record(st)
        if dims.d_ff:
            om.shared_mlp(dims, inp["x"], inp["w_gate_up"], inp["w_down"], y_routed=yr, y=y)
        e[5].record(st)
        torch.cuda.synchronize()
        if i == 0:
            continue
        for k, (a, b) in zip(stages, [(0, 1), (1, 2), (3, 4), (4, 5)]):
            stages[k].append(e[a].elapsed_time(e[b]))
        if sliced:
            passes["a6_pass_z"].append(e[3].elapsed_time(e[6]))
            passes["a6_pass_v"].append(e[6].elapsed_time(e[4]))
    stage_ms = {k: statistics.median(v) for k, v in stages.items()}
    if token or dense:  # the plan was built for the load metrics only; the layer does not schedule
        stage_ms["schedule_a4_a5"] = 0.0
    usage, uneven = om.load_stats(plan).cpu().tolist()  # Expert Usage / Unevenness
    if sliced:
        stage_ms.update({k: statistics.median(v) for k, v in passes.items()})
    n_active = int(plan["n_active"].item())

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        # the public host-buffer call: x from pinned host memory, y back to pinned host
        # memory, both transfers inside the timed region (overlapped with the router and
        # the shared MLP by omnimoe_layer_fwd_host)
        xh = inp["x"].cpu().pin_memory()
        yh = torch.empty(y.shape, dtype=y.dtype).pin_memory()
        xd = torch.empty_like(inp["x"])
        cs = torch.cuda.Stream()

        def host_step():
            om.layer_fwd_host(dims, xh, inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"), inp.get("w_down"),
                              y_host=yh, x_dev=xd, y_dev=y, ws=lws, chunks=args.e2e_chunks, copy_stream=cs)
        for _ in range(2):
            host_step()
        torch.cuda.synchronize()
        tot = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.zero_()
            a.record(st)
            host_step()
            b.record(st)
            torch.cuda.synchronize()
            tot.append(a.elapsed_time(b))
        e2e_ms = statistics.mean(tot)
        eb = 2 if dims.dtype == 0 else 4
        e2e = {"value": L / (e2e_ms / 1000.0), "unit": "tokens/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": L * dims.d * eb, "d2h_bytes_per_step": L * dims.d * eb,
               "api": f"omnimoe_layer_fwd_host ({args.e2e_chunks} chunks)"}

    pk = peaks()
    B = om.group_size(dims)
    eta = M / max(n_active, 1)
    other = {}
    if sliced:
        # the two kernels of the SLICED executor; the dominant one is the roofline
        eb = 2
        zb = n_active * dims.d * eb + L * dims.d * eb + 12 * M + 4 * M              # W rows once, x, plan, a
        vb = n_active * dims.d * eb + 8 * M + 4 * L * dims.d                       # V rows once, pairs, y write
        zl2 = M * dims.d * eb + n_active * dims.d * eb + 12 * M                    # x per task + W + plan
        nbv = om.v_bands(dims, dims.N, L)
        vl2 = M * dims.d * eb + 8 * M * (dims.d // 64) + 4 * L * dims.d * (2 * nbv - 1)  # v pieces + pairs + y
        zk = "expert_zdot256_kernel" if dims.d % 512 == 0 else "expert_zdot_kernel"
        cand = {zk: (zb, zl2, stage_ms["a6_pass_z"], L2_GATHER_GBS["row4k"], 1),
                "expert_vslice_kernel": (vb, vl2, stage_ms["a6_pass_v"], L2_GATHER_GBS["piece128"], nbv)}
        kern = max(cand, key=lambda k: cand[k][2])
        for k, (hb, l2b, kms, l2pk, nl) in cand.items():
            other[k] = {"algorithmic_hbm_bytes": hb, "ms": kms, "launches": nl, "hbm_gbs": hb / kms / 1e6,
                        "hbm_frac": hb / kms / 1e6 / pk["hbm"], "l2_bytes_dataflow": l2b,
                        "l2_gbs": l2b / kms / 1e6, "l2_peak_gbs": l2pk, "l2_frac": l2b / kms / 1e6 / l2pk}
        a6_bytes, l2_bytes, a6_ms, l2_peak, n_launch = cand[kern]
    else:
        kern = "expert_token_kernel" if token else ("expert_group_tma_kernel" if B > 1 else "expert_warp_kernel")
        if dense:
            kern = "gemm_tc_kernel (dense routed branch)"
        a6_bytes, a6_ms = a6_algorithmic_bytes(dims, L, n_active, M), stage_ms["expert_a6"]
        l2_bytes, l2_peak, n_launch = 2 * M * dims.d * 2, L2_GATHER_GBS["row4k"], 1
    a6_gbs = a6_bytes / (a6_ms / 1000.0) / 1e9
    traffic, tsrc = ncu_traffic(w.name, kern)
    if traffic is not None:  # ncu captures one launch; a pass of n_launch band launches moves n_launch x that
        traffic *= n_launch
    if dense:  # two dense GEMMs: the tensor roofline (L x N x d MACs each)
        tf = 2 * 2.0 * L * dims.N * dims.d / (a6_ms / 1000.0) / 1e12
        roofline = {"bound": "tensor", "achieved": tf, "peak": pk["bf16_sus"], "unit": "TFLOP/s",
                    "frac": tf / pk["bf16_sus"], "traffic": None, "kernel": "gemm_tc_kernel x2 (dense routed branch)",
                    "avg_launch_ms": a6_ms, "peak_source": pk["src"] + " bf16 sustained",
                    "note": f"eta = {eta:.0f}: Z = x W^T and y = A V on tcgen05 (DESIGN.md §4.4)",
                    # the method's own work: 2 FLOP per task for z = x.w_e and 2 for y += a v_e, per column
                    "method_work": {"flop": 4.0 * dims.d * M,
                                    "achieved_tflops": 4.0 * dims.d * M / (a6_ms / 1000.0) / 1e12,
                                    "dense_equivalent_flop": 2 * 2.0 * L * dims.N * dims.d,
                                    "note": "the dense GEMMs do L N d MACs each; the method needs 2 d per task"}}
    if not dense:
      roofline = {"bound": "hbm", "achieved": a6_gbs, "peak": pk["hbm"], "unit": "GB/s", "frac": a6_gbs / pk["hbm"],
                "traffic": traffic, "kernel": f"{kern} (a6)", "algorithmic_bytes_per_launch": a6_bytes,
                "avg_launch_ms": a6_ms, "peak_source": pk["src"] + " hbm_gbs (copy)",
                "traffic_source": tsrc,
                "l2": {"bytes_per_launch": l2_bytes, "achieved_gbs": l2_bytes / (a6_ms / 1000.0) / 1e9,
                       "peak_gbs": l2_peak, "frac": l2_bytes / (a6_ms / 1000.0) / 1e9 / l2_peak,
                       "peak_source": "tools/l2_ceiling.cu (profiles/r2/l2_ceiling/l2_ceiling.json)"},
                "note": f"every task moves a d-row of x (pass Z) and of V (pass V) through L2 whatever the loop "
                        f"order (eta = M/|E_active| = {eta:.1f} tasks share an expert, the only reuse); the binding "
                        "roofline is L2 -> SM throughput, not HBM -- DESIGN.md §4.4, profiles/r1/README.md"}
    R_ = dims.n_rows + dims.n_cols
    router_ops = 2.0 * L * dims.n_heads * R_ * dims.d
    mlp_flops = 6.0 * L * dims.d * dims.d_ff
    cpu = parity = None
    if not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        # the timed layer's output and routing on the same inputs, for the parity counters
        yo, io, go = om.layer_fwd(dims, inp["x"], inp["subkeys"], inp["W"], inp["V"], inp.get("w_gate_up"),
                                 inp.get("w_down"), return_routing=True, ws=lws)
        gpu = (yo.float().cpu().numpy(), io.cpu().numpy().reshape(L, -1), go.cpu().numpy().reshape(L, -1))
        del yo, io, go
        rate, done, t, parity = cpu_oracle_rate(w, args.cpu_seconds, 1 << 20, nth, oinp, gpu)
        parity["note"] = ("layer output of the timed call vs oracle.layer on the cpu_baseline sample: router id "
                          "sets per token-head (reading Q10: mismatches allowed only where the oracle's score gap "
                          "< 1e-6), e_tok / e_elt (Q17, bound 1e-2 in bf16)")
        cpu = {"value": rate, "unit": "tokens/s", "cores": nth, "kind": "oracle",
               "sample": f"{done} tokens of {w.name} (oracle layer: exact logits, product top-K, token-centric "
                         f"routed branch, shared MLP): {t:.1f} s of oracle time on {nth} threads"}
    line = {
        "metric": METRIC, "value": L / (ms / 1000.0), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "latency_ms": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded counter-based generator, DESIGN.md §3)",
        "config": _arm_config(w, args, 1),
        "stage_ms": stage_ms, "n_active": n_active, "tasks": M,
        "load": {"expert_usage": usage, "unevenness": uneven,
                 "note": "PAPER:405-410 (paper's full model: usage 100%, unevenness 0.24 with trained routers; "
                         "here seeded random routers)"},
        "step_ms_min_max": [min(step_ms), max(step_ms)],
        "roofline": roofline,
        "a6_kernels": other,
        "other_rooflines": {
            "router_a1_i8": {"tops_int8": 9 * router_ops / 1e12,
                             "note": "9 int8 limb GEMMs of the exact router (DESIGN.md §4.1)"},
            "shared_mlp_a7": {"tflop": mlp_flops / 1e12, "peak_tflops": pk["bf16_sus"],
                              "achieved_tflops": mlp_flops / (stage_ms["shared_mlp_a7_a8"] / 1e3) / 1e12
                              if dims.d_ff else None}},
        "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
        "gpu_launches": launches, "launches_per_step": launches / max(args.steps, 1),
        "clocks": clk.summary(),
        "context": "paper: 6.7 ms OmniMoE vs 73 ms PEER per layer at 4,096 tokens, d=1024, N=102,400, K=4096 on "
                   "A100 (PAPER:368) -- a different shape (config C4)",
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- N > 1
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md)


def bench_multi(args, w, ws, rk, lr):
    """configs[4] (expert-sharded scale-out): the GLOBAL batch of w.L tokens split over
    the ranks (strong scaling), expert rows N/R per rank, NCCL all-to-all dispatch and
    combine."""
    from paper_2602_05711_b200 import distributed as ep, omnimoe as om
    from synth.workloads import make_inputs
    dims, L = w.dims, w.L
    if dims.N % ws or L % ws:
        raise SystemExit(f"N={dims.N} and L={L} must be divisible by {ws} ranks")
    n_per, L_loc = dims.N // ws, L // ws
    inp = make_inputs(dims, L_loc, w.seed, token_begin=rk * L_loc, expert_rows=(rk * n_per, (rk + 1) * n_per))
    oinp = {"W": inp["W"], "V": inp["V"]} if rk == 0 else None  # rows [0, n_per) for the oracle sample
    if dims.v_layout == om.V_SLICED:  # one-time re-layout of this rank's V shard
        inp["V"] = om.pack_v(dims, inp["V"])
        torch.cuda.synchronize()
    ops = ep.LibOps(dims)
    ops.set_mlp(inp.get("w_gate_up"), inp.get("w_down"))
    comm = ep.TorchComm()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    dx = None
    if args.exchange == "device":  # N3: the fused exchange on the NCCL device API
        hk = dims.n_heads * dims.top_k
        dx = ep.DevExchange(dims, row_cap=L, rec_cap=int(1.5 * L * hk / ws) + 4096)

    def step(x=None, marks=None):
        if dx is not None:
            return ep.ep_layer_fwd_dev(ops, dx, inp["x"] if x is None else x, inp["subkeys"], inp["W"], inp["V"],
                                       n_per, marks=marks)
        return ep.ep_layer_fwd(ops, comm, inp["x"] if x is None else x, inp["subkeys"], inp["W"], inp["V"], n_per,
                               marks=marks)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = om.LAUNCHES
    phase = {}
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms_steps = []
        for i in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            evs = {}

            def mark(name):
                e = torch.cuda.Event(enable_timing=True)
                e.record(st)
                evs[name] = e
            step(marks=mark)
            torch.cuda.synchronize()
            names = list(evs)
            ms_steps.append(evs[names[0]].elapsed_time(evs[names[-1]]))
            for a, b in zip(names, names[1:]):
                phase.setdefault(b, []).append(evs[a].elapsed_time(evs[b]))
    launches = om.LAUNCHES - launches0
    t = torch.tensor([statistics.mean(ms_steps)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    phase_ms = {k: statistics.median(v) for k, v in phase.items()}
    # message sizes of one more step: rows / records this rank sent to OTHER ranks (its own
    # block stays local), the bf16 partial rows it sent back; the records it processed
    y_out, rst = ep.ep_layer_fwd(ops, comm, inp["x"], inp["subkeys"], inp["W"], inp["V"], n_per, return_state=True)
    if dx is not None:
        y_out = step()
    torch.cuda.synchronize()
    cnt = ops.last_route  # this rank's routing (that step)
    eb = 2 if dims.dtype == 0 else 4
    sent_rows = sum(c for s_, c in enumerate(rst.send_tok) if s_ != rk)
    sent_recs = sum(c for s_, c in enumerate(rst.send_task) if s_ != rk)
    back_rows = sum(c for s_, c in enumerate(rst.recv_tok) if s_ != rk)
    nvl_bytes = sent_rows * dims.d * eb + sent_recs * 12 + back_rows * dims.d * 2
    a2a_ms = phase_ms.get("all_to_all_dispatch", 0.0) + phase_ms.get("all_to_all_combine", 0.0)
    m_loc, rows_loc = sum(rst.recv_task), sum(rst.recv_tok)
    e2e = None
    if not args.no_e2e:
        xh = inp["x"].cpu().pin_memory()
        xd = torch.empty_like(inp["x"])
        tot = []
        for _ in range(max(2, args.steps)):
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            xd.copy_(xh, non_blocking=True)
            yv = step(xd)
            yh = yv.to("cpu", non_blocking=False)
            b.record(st)
            torch.cuda.synchronize()
            tot.append(a.elapsed_time(b))
        te = torch.tensor([statistics.mean(tot[1:])], dtype=torch.float64, device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": L / (float(te.item()) / 1000.0), "unit": "tokens/s", "ms_per_step": float(te.item()),
               "h2d_bytes_per_step": L * dims.d * eb, "d2h_bytes_per_step": L * dims.d * eb}
        del yh
    if rk == 0:
        pk = peaks()
        exp_ms = phase_ms.get("expert", 0.0)
        import math
        n_act_est = n_per * -math.expm1(-m_loc / n_per)  # E|active experts of the shard| (uniform routing)
        # W and V rows of the active experts once, the received x rows, fp32 partial rows, 24 B per task
        a6_bytes = 2 * n_act_est * dims.d * eb + rows_loc * dims.d * (eb + 4) + 24 * m_loc
        roofline = {"bound": "hbm", "achieved": a6_bytes / (exp_ms / 1e3) / 1e9 if exp_ms else None,
                    "peak": pk["hbm"], "unit": "GB/s",
                    "frac": a6_bytes / (exp_ms / 1e3) / 1e9 / pk["hbm"] if exp_ms else None, "traffic": None,
                    "kernel": "rank 0 expert phase (unpack + schedule + SLICED a6 + bf16 partials)",
                    "algorithmic_bytes_per_launch": a6_bytes, "avg_launch_ms": exp_ms,
                    "peak_source": pk["src"] + " hbm_gbs (copy)",
                    "nvlink": {"bytes_per_step_rank0": nvl_bytes, "a2a_ms": a2a_ms,
                               "achieved_gbs": nvl_bytes / (a2a_ms / 1e3) / 1e9 if a2a_ms else None,
                               "peak_gbs": NVLINK_PEER_GBS,
                               "peak_source": "measured peer copy per direction (B200_PROFILING.md)"}}
        cpu = parity = None
        if not args.no_cpu_baseline:
            nth = os.cpu_count() or 1
            gpu = (y_out.float().cpu().numpy(), cnt[0].cpu().numpy(), cnt[1].cpu().numpy())
            sub_w = dataclasses.replace(w, L=L_loc)
            rate, done, tcpu, parity = cpu_oracle_rate(sub_w, args.cpu_seconds, 1 << 20, nth, None, gpu)
            parity["note"] = "rank 0's tokens: EP layer output vs oracle.layer (reading Q10 / Q17)"
            cpu = {"value": rate, "unit": "tokens/s", "cores": nth, "kind": "oracle",
                   "sample": f"{done} tokens of {w.name} (rank 0's slice): {tcpu:.1f} s of oracle time on {nth} threads"}
        line = {"metric": METRIC, "value": L / (ms / 1000.0), "unit": "tokens/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "latency_ms": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (seeded counter-based generator, DESIGN.md §3)",
                "config": _arm_config(w, args, ws),
                "phase_ms_rank0": phase_ms, "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
                "parity": parity, "gpu_launches": launches, "launches_per_step": launches / max(args.steps, 1),
                "clocks": clk.summary()}
        if args.backend == "gloo":
            line["dry_run"] = ("gloo with host-staged all-to-alls (ranks may share a GPU): a protocol run, "
                               "not an NVLink measurement")
        print(json.dumps(line), flush=True)
    dist.barrier()
    return 0


def _workload(args):
    """The workload of this run: config, V layout (auto: the executor the measurements favour,
    DESIGN.md §4.4), ablation switches."""
    from paper_2602_05711_b200 import configs, omnimoe as om
    w = configs.get(args.config)
    eta = expected_eta(w.dims, w.L)
    # auto: the V layout whose executor the measurements favour -- rows for
    # the token-centric (eta < 2) and dense (K >= N/40) executors, SLICED for 2 <= eta <= 32
    dense_rows = om.layer_executor(w.dims, w.L) == om.EXPERT_DENSE
    sliced = args.expert_kernel == "auto" and (args.v_layout == "sliced" or
                                               (args.v_layout == "auto" and 2.0 <= eta <= 32.0 and not dense_rows))
    w = configs.get(args.config, v_layout=om.V_SLICED if sliced else om.V_ROWS,
                    v_band_bytes=int(args.v_band_mb * (1 << 20)))
    if args.expert_kernel != "auto":
        ek = {"token": om.EXPERT_TOKEN, "warp": om.EXPERT_WARP}[args.expert_kernel]
        w = configs.get(args.config, expert_kernel=ek, group_size=1 if ek == om.EXPERT_WARP else 0)
    if args.router == "dense":
        w = configs.get(w.name, **{k: getattr(w.dims, k) for k in ("v_layout", "expert_kernel", "group_size")},
                        router=om.ROUTER_DENSE)
    if args.no_shared_mlp:
        w = configs.get(w.name, **{k: getattr(w.dims, k) for k in ("v_layout", "expert_kernel", "group_size",
                                                                   "router")}, d_ff=0)
    return w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None,
                    help="workload (default: C3a on one GPU -- configs[2]; C5 over N > 1 GPUs -- configs[4], "
                         "the expert-sharded scale-out, strong scaling)")
    ap.add_argument("--exchange", default="host", choices=["host", "device"],
                    help="N > 1: host (NCCL all_to_all) or device (fused peer stores on the NCCL device API, N3)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="N > 1 process group: nccl (the product), or gloo with host-staged all-to-alls (dry run)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle time of the cpu_baseline sample")
    ap.add_argument("--ref-seconds", type=float, default=60.0, help="total oracle time of --impl reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="token chunks of the host-buffer call")
    ap.add_argument("--router", default="cpr", choices=["cpr", "dense"],
                    help="cpr: the Cartesian Product Router; dense: the paper's 'w/o CPR' ablation")
    ap.add_argument("--no-shared-mlp", action="store_true", help="ablation 'w/o Shared Dense MLP' (d_ff = 0)")
    ap.add_argument("--v-layout", default="auto", choices=["auto", "sliced", "rows"],
                    help="layout of the V table: sliced ([d/32][N][32], the two-pass SLICED executor), rows "
                         "([N][d]: grouped ECS, or token-centric when eta < 2), or auto: sliced for "
                         "2 <= eta <= 32 tasks per active expert, rows otherwise (profiles/r1/README.md)")
    ap.add_argument("--expert-kernel", default="auto", choices=["auto", "token", "warp"],
                    help="a6 executor: auto (grouped ECS), token (the paper's 'w/o ECS' ablation), "
                         "warp (expert-major, B = 1)")
    ap.add_argument("--v-band-mb", type=float, default=0.0,
                    help="SLICED pass V: L2 budget of one band step (dims.v_band_bytes; 0 = library choice)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)
    if args.config is None:
        args.config = "C5" if rank_info()[0] > 1 else "C3a"
    ws, rk, lr = rank_info()
    if args.impl == "reference":  # the oracle arm: the same workload object, nothing on the GPU
        from paper_2602_05711_b200 import build as _b
        _b.build()
        return run_reference(args, _workload(args))
    dev = lr % max(torch.cuda.device_count(), 1)  # (the gloo dry run may put several ranks on one GPU)
    torch.cuda.set_device(dev)
    if ws > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo", init_method="env://")
    from paper_2602_05711_b200 import build, configs
    if rk == 0:
        build.build()
    if ws > 1:
        dist.barrier()
    w = _workload(args)
    try:
        if ws > 1:
            return bench_multi(args, w, ws, rk, lr)
        return bench_single(args, w, lr)
    finally:
        if ws > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
