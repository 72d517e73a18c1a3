"""Decode-sized expert FFN (readme_expert_ffn, one launch) at B tokens over U unique experts (tokens spread
evenly over experts 0..U-1), under knob variants; CUDA-graph replays, L2 flushed, variants alternated.
Measurement only. Usage: python scripts/decode_u_lab.py "k=v:k=v,k=v" [B]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_19123_b200 import readme as rd  # noqa: E402

spec = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
variants = spec.split(",")
H, E, d = 4096, 8, 5504
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")
res = {}
for U in (1, 2, 4, 8):
    x = torch.randn(B, H, device="cuda", generator=g).bfloat16()
    lg = np.full((B, E), -4.0, dtype=np.float32)
    lg[np.arange(B), np.arange(B) % U] = 4.0
    plan = rd.route(torch.from_numpy(lg).cuda(), 1)
    xs = rd.dispatch(x, plan.dest, 1)
    ys = torch.empty_like(xs)
    ws = torch.empty(rd.expert_ffn_workspace_bytes(B, H, E, d, torch.bfloat16), dtype=torch.uint8, device="cuda")
    graphs = {}
    for v in variants:
        kvs = [(kv.split("=")[0], int(kv.split("=")[1])) for kv in v.split(":") if kv]
        for kn, kv in kvs:
            rd.set_knob(kn, kv)
        fn = lambda: rd.expert_ffn(xs, plan.offsets, wg, wu, wd, out=ys, ws=ws)
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        graphs[v] = gr
        for kn, _ in kvs:
            rd.reset_knob(kn)
    ms = {v: [] for v in variants}
    for _ in range(15):
        for v in variants:
            flush.zero_()
            flush_r.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            graphs[v].replay()
            b.record()
            torch.cuda.synchronize()
            ms[v].append(a.elapsed_time(b))
    wbytes = U * 3 * H * d * 2
    for v in variants:
        m = sorted(ms[v])[3:-3]
        t = sum(m) / len(m)
        res.setdefault(U, {})[v] = {"us": round(t * 1e3, 1), "weights_GBps": round(wbytes / (t * 1e-3) / 1e9)}
print(json.dumps({"B": B, "results": res}))
