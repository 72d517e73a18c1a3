"""Timeline of one readme_moe_layer step (config 2) from the kernels' %globaltimer trace
(readme_debug_trace): when the FFN gets past its prologue and starts its first gate/up tile relative to the
route and the dispatch. Measurement only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

T, H, E, d = int(os.environ.get("TRACE_T", "8192")), 4096, 8, 5504
K = int(os.environ.get("TRACE_K", "1"))
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
lg = torch.from_numpy(synth.router_logits(T, E, seed=3)).cuda()
plan = rd.new_plan(T, E, K, "cuda")
ws = torch.empty(rd.moe_layer_workspace_bytes(T, H, E, d, K, torch.bfloat16), dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
tr = torch.zeros(16, dtype=torch.int64, device="cuda")
MAXU = -1  # all ones as int64


def run():
    rd.moe_layer(x, wg, wu, wd, k=K, logits=lg, plan=plan, out=y, ws=ws)


GRAPH = os.environ.get("TRACE_GRAPH", "1") == "1"
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd.lib().readme_debug_trace(tr.data_ptr())  # kernels read the buffer pointer at launch (captured below)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        run()
torch.cuda.synchronize()
if GRAPH:
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        run()
    run = gr.replay  # noqa: F811
res = []
for it in range(5):
    tr.zero_()
    for i in (0, 2, 3, 5):
        tr[i] = MAXU
    flush.fill_(it)
    st = torch.cuda.current_stream().cuda_stream
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rd.lib().readme_debug_mark(8, st)
    run()
    rd.lib().readme_debug_mark(9, st)
    b.record()
    torch.cuda.synchronize()
    ev_us = a.elapsed_time(b) * 1e3
    v = [int(a) & ((1 << 64) - 1) for a in tr.tolist()]
    t0 = v[5]
    res.append({"route_end": (v[6] - t0) / 1e3, "dispatch_start": (v[0] - t0) / 1e3, "dispatch_end": (v[1] - t0) / 1e3,
                "ffn_past_prologue": (v[2] - t0) / 1e3, "ffn_first_tile_ready": (v[3] - t0) / 1e3,
                "ffn_end": (v[4] - t0) / 1e3, "mark_before": (v[8] - t0) / 1e3, "mark_after": (v[9] - t0) / 1e3,
                "event_us": ev_us})
rd.lib().readme_debug_trace(None)
print(json.dumps({"mode": os.environ.get("README_ROUTE", "default"), "graph": GRAPH, "us_from_route_start": res},
                 indent=0))
