"""Serving MoE layers from host memory with the copies overlapped (the e2e path): batches live in pinned
host buffers; each batch's tokens and logits go host->device on a copy stream, the layer runs on the
compute stream (readme_moe_layer: route + dispatch + grouped expert FFN + combine), and the result goes
device->host on a second copy stream. Device buffers are double-buffered and ordered with CUDA events, so
while batch i computes, batch i+1 uploads and batch i-1 downloads (PCIe is full duplex): the steady-state
step costs max(H2D, compute, D2H) instead of their sum. Every byte of every batch still crosses PCIe.
"""
from __future__ import annotations

import torch

from . import readme as rd


class HostPipeline:
    def __init__(self, T: int, H: int, E: int, k: int, w_gate, w_up, w_down, logits_dtype=torch.float32,
                 nbuf: int = 2, device=None):
        dev = torch.device(device) if device is not None else w_gate.device
        self.dev, self.k, self.w = dev, k, (w_gate, w_up, w_down)
        dt = w_gate.dtype
        d = w_gate.shape[1]
        self.nbuf = nbuf
        self.x = [torch.empty((T, H), dtype=dt, device=dev) for _ in range(nbuf)]
        self.lg = [torch.empty((T, E), dtype=logits_dtype, device=dev) for _ in range(nbuf)]
        self.y = [torch.empty((T, H), dtype=dt, device=dev) for _ in range(nbuf)]
        self.plan = [rd.new_plan(T, E, k, dev) for _ in range(nbuf)]
        self.ws = [torch.empty(rd.moe_layer_workspace_bytes(T, H, E, d, k, dt), dtype=torch.uint8, device=dev)
                   for _ in range(nbuf)]
        self.up = torch.cuda.Stream(device=dev)
        self.down = torch.cuda.Stream(device=dev)

    def run(self, xs_host, lgs_host, ys_host, compute_stream=None):
        """xs_host[i] / lgs_host[i] (pinned) -> ys_host[i] (pinned), for every i; returns the streams' last
        events (the caller synchronises)."""
        comp = compute_stream or torch.cuda.current_stream(self.dev)
        n = len(xs_host)
        uploaded = [None] * self.nbuf   # x/lg of buffer b are on the device
        computed = [None] * self.nbuf   # y of buffer b is ready; x/lg of b are free again
        downloaded = [None] * self.nbuf  # y of buffer b has reached the host
        for i in range(n):
            b = i % self.nbuf
            with torch.cuda.stream(self.up):
                if computed[b] is not None:
                    self.up.wait_event(computed[b])
                self.x[b].copy_(xs_host[i], non_blocking=True)
                self.lg[b].copy_(lgs_host[i], non_blocking=True)
                uploaded[b] = torch.cuda.Event()
                uploaded[b].record(self.up)
            comp.wait_event(uploaded[b])
            if downloaded[b] is not None:
                comp.wait_event(downloaded[b])
            with torch.cuda.stream(comp):
                rd.moe_layer(self.x[b], *self.w, k=self.k, logits=self.lg[b], plan=self.plan[b], out=self.y[b],
                             ws=self.ws[b])
                computed[b] = torch.cuda.Event()
                computed[b].record(comp)
            with torch.cuda.stream(self.down):
                self.down.wait_event(computed[b])
                ys_host[i].copy_(self.y[b], non_blocking=True)
                downloaded[b] = torch.cuda.Event()
                downloaded[b].record(self.down)
        return downloaded
