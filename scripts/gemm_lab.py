"""GEMM experiments (not the product path): time readme_expert_gate_up / readme_expert_down under variants
selected by env knobs, on config-2 shapes with (a) the bench's routing and (b) perfectly balanced
1024-row experts. Prints one JSON line per variant."""
import json
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2410_19123_b200 import readme as rd  # noqa: E402

dev = torch.device("cuda", 0)
T, H, d, E = 8192, 4096, 5504, 8
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
wg, wu, wd = synth.expert_weights_device(E, d, H, dev, seed=5)
xs = synth.to_torch(synth.tokens(T, H, seed=6), "bf16").to(dev)
h = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
ys = torch.empty((T, H), dtype=torch.bfloat16, device=dev)
lg = synth.router_logits(T, E, seed=synth.MASTER_SEED + 2)
counts = np.bincount(lg.argmax(1), minlength=E)
offs = {"bench": np.concatenate([[0], np.cumsum(counts)]).astype(np.int32),
        "balanced": (np.arange(E + 1) * (T // E)).astype(np.int32)}


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


variant = os.environ.get("README_LAB", "0") + "/" + os.environ.get("README_FFN_KERNEL", "2cta")
for name, off in offs.items():
    o = torch.from_numpy(off).to(dev)
    gu = timeit(lambda: rd.expert_gate_up(xs, o, wg, wu, out=h))
    dn = timeit(lambda: rd.expert_down(h, o, wd, out=ys))
    ws = torch.empty(rd.expert_ffn_workspace_bytes(T, H, E, d, torch.bfloat16), dtype=torch.uint8, device=dev)
    ffn = timeit(lambda: rd.expert_ffn(xs, o, wg, wu, wd, out=ys, ws=ws))
    print(json.dumps({"variant": variant, "routing": name, "gate_up_ms": gu, "down_ms": dn, "expert_ffn_ms": ffn,
                      "gate_up_tflops": 4 * T * H * d / gu / 1e9, "down_tflops": 2 * T * H * d / dn / 1e9,
                      "expert_ffn_tflops": 6 * T * H * d / ffn / 1e9}), flush=True)
