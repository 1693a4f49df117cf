"""B200-native OmniMoE atomic-expert layer forward (arXiv 2602.05711).

The product is libomnimoe.so (C ABI in include/omnimoe.h); this package is its
thin Python binding (``omnimoe``), the workload configurations (``configs``)
and the multi-GPU expert-parallel orchestration (``distributed``).
"""
from . import configs  # noqa: F401
from .omnimoe import (BF16, F32, SILU, IDENTITY, LayerDims, OmniMoEError, expert_fwd,  # noqa: F401
                      gemm_bf16, layer_fwd, load, route, router_logits, schedule, shared_mlp,
                      workspace, workspace_size)
