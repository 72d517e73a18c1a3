"""Expert FFN alone (readme_expert_ffn, one ffn_layer2 launch) at several batch sizes under library knob
variants (readme_debug_set_knob; e.g. ffn_swap=0,64 or ffn_mt=128,256), CUDA-graph replays, L2 flushed
before each, variants alternated round by round on the same box. Measurement only.
Usage: python scripts/ffn_lab.py KNOB=a,b [T1 T2 ...]
       python scripts/ffn_lab.py "k1=a:k2=b,k1=c" [T ...]   (each comma-separated variant sets one or more knobs)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

spec = sys.argv[1]
if ":" in spec or spec.count("=") > 1:  # variants of several knobs each
    vals = [v for v in spec.split(",")]
    var = "variants"
    settings = {v: [(kv.split("=")[0], int(kv.split("=")[1])) for kv in v.split(":")] for v in vals}
else:
    var, vv = spec.split("=")
    vals = [int(v) for v in vv.split(",")]
    settings = {v: [(var, v)] for v in vals}
Ts = [int(t) for t in sys.argv[2:]] or [256, 512, 1024, 2048, 4096, 8192]
H, E, d = 4096, 8, 5504
g = torch.Generator(device="cuda").manual_seed(1)
wg = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wu = (torch.randn(E, d, H, device="cuda", generator=g) / 64).bfloat16()
wd = (torch.randn(E, H, d, device="cuda", generator=g) / 74).bfloat16()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")  # read after the write: no dirty lines left
res = {}
for T in Ts:
    x = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    # the bench's routing logits at T = 8192 (config 2 counts), else seeded by T
    seed = synth.MASTER_SEED + 2 if T == 8192 else T
    plan = rd.route(torch.from_numpy(synth.router_logits(T, E, seed=seed)).cuda(), 1)
    xs = rd.dispatch(x, plan.dest, 1)
    ys = torch.empty_like(xs)
    ws = torch.empty(rd.expert_ffn_workspace_bytes(T, H, E, d, torch.bfloat16), dtype=torch.uint8, device="cuda")
    graphs = {}
    for v in vals:
        for kn, kv in settings[v]:
            rd.set_knob(kn, kv)
        fn = lambda: rd.expert_ffn(xs, plan.offsets, wg, wu, wd, out=ys, ws=ws)
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        graphs[v] = gr
        for kn, _ in settings[v]:
            rd.reset_knob(kn)
    ms = {v: [] for v in vals}
    for _ in range(15):
        for v in vals:
            flush.zero_()
            flush_r.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            graphs[v].replay()
            b.record()
            torch.cuda.synchronize()
            ms[v].append(a.elapsed_time(b))
    for v in vals:
        m = sorted(ms[v])[3:-3]
        t = sum(m) / len(m)
        res.setdefault(T, {})[v] = {"us": round(t * 1e3, 1), "TFLOPs": round(6 * T * H * d / (t * 1e-3) / 1e12, 1)}
print(json.dumps({"knob": var, "counts_T8192": plan.counts.tolist() if Ts[-1] == 8192 else None, "results": res}))
