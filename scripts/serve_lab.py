"""Per-step GPU times of the serving simulation (expert-aware vs FIFO) at config-3 shape. Measurement only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_19123_b200 import serving  # noqa: E402

H, E, d = 4096, 8, 5504
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
for rep in range(2):
    for pol in ("expert_aware", "fifo"):
        r = serving.simulate(pol, wg, wu, wd, steps=24)
        print(rep, pol, r["mean_unique_experts"], round(r["mean_step_ms"], 4))
