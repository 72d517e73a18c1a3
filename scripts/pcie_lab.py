"""PCIe copy rates on this box (pinned host memory): H2D alone, D2H alone, both at once on two streams;
64 MiB per copy (a config-2 batch of bf16 rows). Measurement only."""
import json

import torch

N = 64 << 20
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def rate(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(up):
        d_in.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(up)


def d2h():
    with torch.cuda.stream(down):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(down)


def both():
    with torch.cuda.stream(up):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(down):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(up)
    torch.cuda.current_stream().wait_stream(down)


def chunked_both(nchunk=8):
    c = N // nchunk
    for i in range(nchunk):
        with torch.cuda.stream(up):
            d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
        with torch.cuda.stream(down):
            h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
    torch.cuda.current_stream().wait_stream(up)
    torch.cuda.current_stream().wait_stream(down)


res = {}
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("both_chunked8", chunked_both)):
    ms = rate(fn)
    res[name] = {"ms": round(ms, 4), "GBps_each_direction": round(N / (ms * 1e-3) / 1e9, 1)}
print(json.dumps(res))
