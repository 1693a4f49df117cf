"""Workload configurations (BASELINE.json configs, made concrete in SURVEY.md 8.0;
readings Q2-Q5 in DESIGN.md)."""
from __future__ import annotations

from dataclasses import dataclass, replace

from .omnimoe import BF16, LayerDims


@dataclass(frozen=True)
class Workload:
    name: str
    dims: LayerDims
    L: int
    seed: int
    note: str = ""


def _w(name, d, nr, nc, K, h, L, dff, seed, note=""):
    return Workload(name, LayerDims(d=d, n_rows=nr, n_cols=nc, top_k=K, n_heads=h, d_ff=dff, dtype=BF16),
                    L, seed, note)


CONFIGS = {
    # BASELINE.json configs[0]: tiny CPU-checkable layer
    "C1": _w("C1", 64, 32, 32, 8, 1, 256, 128, 0, "tiny CPU-checkable layer (configs[0])"),
    # configs[1]: router-only sweep
    "C2": _w("C2", 1024, 256, 256, 16, 4, 8192, 0, 1, "router-only sweep (configs[1])"),
    # configs[2]: paper-shaped layer on 1 GPU (K=512, h=1 per reading Q4; d_ff = d per Q2)
    "C3a": _w("C3a", 2048, 1024, 1024, 512, 1, 16384, 2048, 2, "paper-shaped layer, K=512 (configs[2])"),
    "C3b": _w("C3b", 2048, 1024, 1024, 16, 1, 16384, 2048, 2, "paper-shaped layer, K=16 (configs[2], HBM-bound regime)"),
    # configs[3]: the 6.7 ms comparison shape (reading Q5) and protocol-consistent neighbours
    "C4": _w("C4", 1024, 320, 320, 4096, 1, 4096, 1024, 3, "6.7 ms shape (configs[3])"),
    "C4p": _w("C4p", 1024, 320, 320, 4096, 1, 1024, 1024, 3, "K=4096, 1K tokens"),
    "C4pp": _w("C4pp", 1024, 320, 320, 512, 1, 4096, 1024, 3, "K=512, 4K tokens"),
    # configs[4]: expert-sharded scale-out (global sizes; per-rank tokens L/R)
    "C5": _w("C5", 2048, 2048, 2048, 512, 1, 65536, 2048, 1, "expert-sharded scale-out (configs[4])"),
    "C5s": _w("C5s", 2048, 2048, 2048, 16, 1, 65536, 2048, 1, "scale-out, K=16"),
}


def get(name: str, **over) -> Workload:
    w = CONFIGS[name]
    if over:
        dims_over = {k: v for k, v in over.items() if hasattr(w.dims, k)}
        rest = {k: v for k, v in over.items() if not hasattr(w.dims, k)}
        w = replace(w, dims=replace(w.dims, **dims_over), **rest)
    return w
