"""HostPipeline (e2e: pinned host batches in and out) at config-2 shape with 2/3/4 device buffer sets.
Measurement only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200.pipeline import HostPipeline  # noqa: E402

T, H, E, d, K = 8192, 4096, 8, 5504, 12
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
x_h = [torch.randn(T, H, generator=torch.Generator().manual_seed(i)).bfloat16().pin_memory() for i in range(2)]
lg_h = [torch.from_numpy(synth.router_logits(T, E, seed=i)).pin_memory() for i in range(2)]
out = {}
for nbuf in (2, 3, 4):
    pipe = HostPipeline(T, H, E, 1, wg, wu, wd, nbuf=nbuf)
    ys = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(nbuf)]
    xs, ls = [x_h[i % 2] for i in range(K)], [lg_h[i % 2] for i in range(K)]
    pipe.run(xs[:nbuf], ls[:nbuf], ys)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.up)
        last = pipe.run(xs, ls, [ys[i % nbuf] for i in range(K)])
        for ev in last:
            if ev is not None:
                pipe.down.wait_event(ev)
        b.record(pipe.down)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / K)
    out[nbuf] = {"ms_per_batch": round(best, 4), "Mtok_s": round(T / best / 1e3, 3)}
print(json.dumps(out))
