"""Route micro-benchmark: readme_route alone, CUDA-graph replays of 50 calls, per batch size and
implementation (README_ROUTE / README_ROUTE_CLUSTER set by the caller)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

out = {}
for T in (256, 2048, 8192, 65536):
    lg = torch.from_numpy(synth.router_logits(T, 8, seed=T)).cuda()
    plan = rd.new_plan(T, 8, 1, "cuda")
    ws = torch.empty(rd.route_workspace_bytes(T, 8, 1), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            rd.route(lg, 1, plan=plan, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(50):
            rd.route(lg, 1, plan=plan, ws=ws)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 50 * 1e3)
    out[T] = round(best, 2)
print(json.dumps({"impl": os.environ.get("README_ROUTE", "default"),
                  "cluster": os.environ.get("README_ROUTE_CLUSTER", "auto"), "us_per_route": out}))
