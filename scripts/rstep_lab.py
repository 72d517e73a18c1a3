"""readme_router_step alone at the config-3 shape (256 decode tokens, histories uniform in [0, 4096)), for ncu."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

RW = {kk: synth.to_torch(v, "bf16").cuda() for kk, v in synth.router_weights(n_experts=8, seed=31).items()}
cache = rd.new_router_cache(256, 4096, "cuda")
pos = torch.from_numpy(synth.rng(32, 0).integers(0, 4096, size=256).astype(np.int32)).cuda()
tok = torch.from_numpy(synth.token_ids(256, seed=33)).cuda()
slots = torch.arange(256, dtype=torch.int32, device="cuda")
for _ in range(3):
    rd.router_step(tok, slots, pos, cache, RW)
torch.cuda.synchronize()
