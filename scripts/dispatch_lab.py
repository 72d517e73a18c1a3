"""readme_dispatch alone (scatter form; LAB_OP=combine: readme_combine, k = 1 gather) at T rows x H = 4096
bf16 under library knob variants (readme_debug_set_knob, e.g. dispatch_bulk=0,1), CUDA-graph replays, L2
flushed before each; GB/s = 2 * rows * H * 2 / time. Measurement only.
Usage: python scripts/dispatch_lab.py KNOB=a,b [T1 T2 ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

var, vals = sys.argv[1].split("=")
vals = vals.split(",")
Ts = [int(t) for t in sys.argv[2:]] or [4096, 16384, 65536]
H, E = 4096, 8
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for T in Ts:
    x = torch.randn(T, H, device="cuda").bfloat16()
    plan = rd.route(torch.from_numpy(synth.router_logits(T, E, seed=T)).cuda(), 1)
    xs = torch.empty_like(x)
    ref = None
    for v in vals:
        rd.set_knob(var, int(v))
        if os.environ.get("LAB_OP") == "combine":
            fn = lambda: rd.combine(x, plan.dest, None, 1, out=xs)
        else:
            fn = lambda: rd.dispatch(x, plan.dest, 1, out=xs)
        fn()
        torch.cuda.synchronize()
        if ref is None:
            ref = xs.clone()
        assert torch.equal(ref, xs), f"{var}={v}: result differs"
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        ms = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        ms.sort()
        t = ms[len(ms) // 2]
        res.setdefault(str(T), {})[v] = {"us": round(t * 1e3, 1), "GBps": round(2 * T * H * 2 / (t * 1e-3) / 1e9, 0)}
print(json.dumps({"var": var, "results": res}))
