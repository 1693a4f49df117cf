"""CPU-side checks of the boundary (-m "not gpu"): the C-ABI library builds for
sm_100a, loads, and exports every symbol include/omnimoe.h declares; the
product path never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_05711_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def _declared():
    hdr = open(os.path.join(ROOT, "include", "omnimoe.h")).read()
    return sorted(set(re.findall(r"\b(omnimoe_[a-z_0-9]+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("omnimoe_route", "omnimoe_schedule", "omnimoe_expert_fwd", "omnimoe_layer_fwd",
              "omnimoe_workspace_size", "omnimoe_status_string", "omnimoe_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in _declared():
        assert hasattr(lib, n), n
    from paper_2602_05711_b200 import omnimoe as om
    assert set(om.EXPORTS) <= set(_declared())


def test_sm100a_code_only(lib):
    from paper_2602_05711_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass  # tcgen05 bf16 MMA + TMA in the GEMM engine
    assert "UTCIMMA" in sass  # tcgen05 kind::i8 MMA of the exact router logits


def test_host_side_validation_without_gpu(lib):
    from paper_2602_05711_b200 import omnimoe as om
    om.load()
    d = om.LayerDims(d=64, n_rows=4, n_cols=4, top_k=17)
    with pytest.raises(om.OmniMoEError, match="SHAPE"):
        om.workspace_size(d, 10, om.WS_LAYER)
    d = om.LayerDims(d=60, n_rows=4, n_cols=4, top_k=2)
    with pytest.raises(om.OmniMoEError, match="INVALID_ARGUMENT"):
        om.workspace_size(d, 10, om.WS_ROUTE)
    ok = om.LayerDims(d=64, n_rows=32, n_cols=32, top_k=8, d_ff=128)
    assert om.workspace_size(ok, 256, om.WS_LAYER) > om.workspace_size(ok, 256, om.WS_ROUTE) > 0
    assert lib.omnimoe_status_string  # symbol resolves
    sl = om.LayerDims(d=64, n_rows=32, n_cols=32, top_k=8, d_ff=128, v_layout=om.V_SLICED)
    assert om.workspace_size(sl, 256, om.WS_LAYER) > om.workspace_size(ok, 256, om.WS_LAYER)
    with pytest.raises(om.OmniMoEError, match="UNSUPPORTED"):  # SLICED layout needs d % 64 == 0
        om.workspace_size(om.LayerDims(d=72, n_rows=4, n_cols=4, top_k=2, v_layout=om.V_SLICED), 8, om.WS_LAYER)
    with pytest.raises(om.OmniMoEError, match="INVALID_ARGUMENT"):  # and runs the SLICED executor only
        om.workspace_size(om.LayerDims(d=64, n_rows=4, n_cols=4, top_k=2, expert_kernel=om.EXPERT_GROUP,
                                       v_layout=om.V_SLICED), 8, om.WS_LAYER)
    # dims.flags: OMNIMOE_FLAG_ACT_BF16 is the only defined bit
    assert om.workspace_size(om.LayerDims(d=64, n_rows=4, n_cols=4, top_k=2, flags=om.FLAG_ACT_BF16), 8,
                             om.WS_EXPERT) > 0
    with pytest.raises(om.OmniMoEError, match="INVALID_ARGUMENT"):
        om.workspace_size(om.LayerDims(d=64, n_rows=4, n_cols=4, top_k=2, flags=2), 8, om.WS_EXPERT)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_05711_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "oracle.cpp" not in src and "liboracle" not in src, f


def test_oracle_includes_no_cuda():
    src = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    incs = re.findall(r"^\s*#\s*include\s*[<\"]([^>\"]+)", src, re.M)
    assert incs and not any("cuda" in i.lower() or "omnimoe" in i or "csrc" in i for i in incs), incs


def test_ep_device_library_exports():
    """libomnimoe_ep.so (the NCCL device-API exchange, N3) builds and exports what
    include/omnimoe_ep.h declares; it is a separate library (libomnimoe.so has no NCCL)."""
    from paper_2602_05711_b200 import build
    path = build.build_ep()
    ep = ctypes.CDLL(path)
    hdr = open(os.path.join(ROOT, "include", "omnimoe_ep.h")).read()
    names = sorted(set(re.findall(r"\b(omnimoe_ep_[a-z_0-9]+)\s*\(", hdr)))
    assert "omnimoe_ep_dev_dispatch" in names and "omnimoe_ep_dev_return" in names
    for n in names:
        assert hasattr(ep, n), n
    assert ep.omnimoe_ep_dev_unique_id_bytes() == 128
    out = subprocess.run(["ldd", build.LIB], capture_output=True, text=True).stdout
    assert "nccl" not in out
