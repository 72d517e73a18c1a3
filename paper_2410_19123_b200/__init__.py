"""paper_2410_19123_b200 — B200-native hot path of READ-ME's pre-gated MoE layer (arXiv 2410.19123).

The product is the C-ABI library libreadme_b200.so (include/readme.h) built from csrc/ for sm_100a;
`readme` is its thin Python binding and `ep` composes it with torch.distributed for expert parallelism.
"""
from . import readme  # noqa: F401
from .readme import (Plan, build_experts, combine, dispatch, expert_ffn, moe_layer,  # noqa: F401
                     new_plan, route)

__all__ = ["readme", "Plan", "route", "dispatch", "expert_ffn", "combine", "moe_layer", "build_experts",
           "new_plan"]
