"""paper_2410_19123_b200 — B200-native hot path of READ-ME's pre-gated MoE layer (arXiv 2410.19123).

The product is the C-ABI library libreadme_b200.so (include/readme.h) built from csrc/ for sm_100a;
`readme` is its thin Python binding and `ep` composes it with torch.distributed for expert parallelism.
"""
from . import readme  # noqa: F401
from .readme import (Plan, build_experts, combine, dispatch, expert_down, expert_ffn,  # noqa: F401
                     expert_gate_up, moe_layer, new_plan, route)

__all__ = ["readme", "Plan", "route", "dispatch", "expert_ffn", "expert_gate_up", "expert_down", "combine", "moe_layer", "build_experts",
           "new_plan"]
