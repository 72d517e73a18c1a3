"""readme_router_forward at the config-4 shape (4 requests x 4096 tokens) under library knob variants
(e.g. router_attn=0,1), CUDA-graph replays, L2 flushed (write + read) before each, alternated round by round.
Measurement only. Usage: python scripts/router_lab.py KNOB=a,b"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

var, vals = sys.argv[1].split("=")
vals = [int(v) for v in vals.split(",")]
T, E = 16384, 8
W = {k: synth.to_torch(v, "bf16").cuda() for k, v in synth.router_weights(n_experts=E, seed=7).items()}
ids = torch.from_numpy(synth.token_ids(T, seed=7)).cuda()
starts = torch.arange(0, T + 1, 4096, dtype=torch.int32, device="cuda")
out = torch.empty((T, E), dtype=torch.float32, device="cuda")
ws = torch.empty(rd.router_workspace_bytes(T, 4), dtype=torch.uint8, device="cuda")
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fr = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")
graphs, outs = {}, {}
for v in vals:
    rd.set_knob(var, v)
    fn = lambda: rd.router_forward(ids, starts, W, out=out, ws=ws)
    fn()
    torch.cuda.synchronize()
    outs[v] = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    graphs[v] = g
rd.reset_knob(var)
ms = {v: [] for v in vals}
for _ in range(10):
    for v in vals:
        fw.zero_()
        fr.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graphs[v].replay()
        b.record()
        torch.cuda.synchronize()
        ms[v].append(a.elapsed_time(b))
res = {v: round(sorted(ms[v])[len(ms[v]) // 2], 4) for v in vals}
d = (outs[vals[0]] - outs[vals[-1]]).abs().max().item()
print(json.dumps({"knob": var, "router_forward_ms_median": res, "max_abs_logit_diff_first_vs_last": d}))
