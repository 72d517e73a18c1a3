"""HostPipeline timeline at config-2 shape: per batch, when its upload, layer and download ended (CUDA events,
ms from the start), plus the copies alone in the same pattern. Measurement only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402
from paper_2410_19123_b200.pipeline import HostPipeline  # noqa: E402

T, H, E, d, K = 8192, 4096, 8, 5504, 10
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
x_h = [torch.randn(T, H, generator=torch.Generator().manual_seed(i)).bfloat16().pin_memory() for i in range(2)]
lg_h = [torch.from_numpy(synth.router_logits(T, E, seed=i)).pin_memory() for i in range(2)]
out = {}
pipe = HostPipeline(T, H, E, 1, wg, wu, wd, nbuf=2)
ys = [torch.empty(T, H, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
xs, ls = [x_h[i % 2] for i in range(K)], [lg_h[i % 2] for i in range(K)]


def run_traced(compute=True):
    comp = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(pipe.up)
    evs = []
    for i in range(K):
        b = i % 2
        e_up, e_c, e_dn = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        with torch.cuda.stream(pipe.up):
            if i >= 2:
                pipe.up.wait_event(evs[i - 2][1])
            pipe.x[b].copy_(xs[i], non_blocking=True)
            pipe.lg[b].copy_(ls[i], non_blocking=True)
            e_up.record(pipe.up)
        comp.wait_event(e_up)
        if i >= 2:
            comp.wait_event(evs[i - 2][2])
        if compute:
            rd.moe_layer(pipe.x[b], wg, wu, wd, k=1, logits=pipe.lg[b], plan=pipe.plan[b], out=pipe.y[b], ws=pipe.ws[b])
        e_c.record(comp)
        with torch.cuda.stream(pipe.down):
            pipe.down.wait_event(e_c)
            ys[b].copy_(pipe.y[b], non_blocking=True)
            e_dn.record(pipe.down)
        evs.append((e_up, e_c, e_dn))
    torch.cuda.synchronize()
    return [[round(t0.elapsed_time(e), 3) for e in tr] for tr in evs]


for _ in range(2):
    run_traced()
out["pipeline"] = run_traced()
out["copies_only_pattern"] = run_traced(compute=False)
# the layer alone, back to back
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(K):
    rd.moe_layer(pipe.x[i % 2], wg, wu, wd, k=1, logits=pipe.lg[i % 2], plan=pipe.plan[i % 2], out=pipe.y[i % 2],
                 ws=pipe.ws[i % 2])
b.record()
torch.cuda.synchronize()
out["layer_ms"] = a.elapsed_time(b) / K
# H2D alone, D2H alone, both at once
def t(fn, n=5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    a.record(); [fn() for _ in range(n)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
out["h2d_ms"] = t(lambda: pipe.x[0].copy_(x_h[0], non_blocking=True))
out["d2h_ms"] = t(lambda: ys[0].copy_(pipe.y[0], non_blocking=True))
print(json.dumps(out))
