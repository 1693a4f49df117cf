"""Build libomnimoe.so (sm_100a) and synth/libsynth.so in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libomnimoe.so")
SYNTH_SRC = os.path.join(ROOT, "synth", "synth.cu")
SYNTH_LIB = os.path.join(ROOT, "synth", "libsynth.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


LIB_MEASURE = os.path.join(PKG, "libomnimoe_measure.so")


def build(force: bool = False, verbose: bool = False, measure: bool = False) -> str:
    """measure: the measurement build (-DOMNIMOE_MEASURE, csrc/tuning.cuh) into
    libomnimoe_measure.so -- tools/ sweeps load it with OMNIMOE_LIB=<path>; the product
    library never reads the environment."""
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "omnimoe.h")]
    lib = LIB_MEASURE if measure else LIB
    if force or _stale(lib, deps):
        cmd = [NVCC, *ARCH, *FLAGS, *(["-DOMNIMOE_MEASURE"] if measure else []), "-o", lib, *srcs]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    build_ep(force)
    if force or _stale(SYNTH_LIB, [SYNTH_SRC]):
        subprocess.check_call([NVCC, *ARCH, *FLAGS, "-o", SYNTH_LIB, SYNTH_SRC])
    return lib


EP_SRC = os.path.join(CSRC, "nccl", "ep_dev.cu")
EP_LIB = os.path.join(PKG, "libomnimoe_ep.so")


def nccl_dirs():
    """The NCCL 2.28 headers (with the device API) and library torch uses."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    base = list(spec.submodule_search_locations)[0] if spec else ""
    return os.path.join(base, "include"), os.path.join(base, "lib")


def build_ep(force: bool = False) -> str:
    """libomnimoe_ep.so: the fused expert-parallel exchange on the NCCL device API
    (include/omnimoe_ep.h), linked against torch's libnccl.so.2."""
    inc, lib = nccl_dirs()
    if force or _stale(EP_LIB, [EP_SRC, os.path.join(ROOT, "include", "omnimoe_ep.h")]):
        subprocess.check_call([NVCC, *ARCH, *FLAGS, "-I" + inc, "-o", EP_LIB, EP_SRC, "-L" + lib, "-l:libnccl.so.2",
                               "-Xlinker", "-rpath=" + lib])
    return EP_LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, measure="--measure" in sys.argv))
