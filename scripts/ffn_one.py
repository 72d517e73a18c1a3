"""One expert-FFN configuration (readme_expert_ffn) launched a few times at config-2 shape for ncu: knobs as
NAME=VALUE arguments, rows as the first argument. Measurement only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

T = int(sys.argv[1])
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    rd.set_knob(k, int(v))
H, E, d = 4096, 8, 5504
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
plan = rd.route(torch.from_numpy(synth.router_logits(T, E, seed=synth.MASTER_SEED + 2)).cuda(), 1)
xs = rd.dispatch(x, plan.dest, 1)
ys = torch.empty_like(xs)
ws = torch.empty(rd.expert_ffn_workspace_bytes(T, H, E, d, torch.bfloat16), dtype=torch.uint8, device="cuda")
for _ in range(4):
    rd.expert_ffn(xs, plan.offsets, wg, wu, wd, out=ys, ws=ws)
torch.cuda.synchronize()
