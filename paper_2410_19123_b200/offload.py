"""Memory-constrained mode (NEXT-4 of SURVEY §8(f); §4.1): the experts of L layers live in
pinned host memory and only `capacity` expert slots fit on the device.

Pre-gating decides every token's expert before the backbone runs, so the whole reference
string of (layer, expert) accesses of a batch is known at the outset. That enables
  * fine-grained prefetching: "while computing the i-th layer's forward path in the compute stream, we load
    the i+1-st layer's experts in a separate loading stream", and
  * the Belady-inspired cache: evict the resident expert whose next use is farthest, with the
    exact future from the routing plan (native readme_cache_*).

Compute runs in the library's kernels: the pre-norm dispatch (readme_dispatch_rmsnorm) and the expert FFN
over the slot pools (readme_expert_ffn_slots, expert e -> slot table), with the residual update
x <- x + MoE_l(RMSNorm(x)) fused into the down projection's epilogue. Copies are cudaMemcpyAsync from pinned
memory on the loading stream; CUDA events order "slot loaded" before the layer that reads it and "layer
done" before a copy that overwrites one of its slots.
"""
from __future__ import annotations

import numpy as np
import torch

from . import readme as rd


class OffloadedStack:
    def __init__(self, layers_host, capacity: int, policy: str, device, eps: float = 1e-5):
        self.layers = layers_host          # [(w_gate [E,d,H], w_up, w_down [E,H,d]) pinned CPU bf16]
        self.L = len(layers_host)
        self.E, self.d, self.H = layers_host[0][0].shape
        self.cap = capacity
        self.policy = policy
        self.dev = torch.device(device)
        self.eps = eps
        kw = dict(dtype=torch.bfloat16, device=self.dev)
        self.pool_g = torch.empty((capacity, self.d, self.H), **kw)
        self.pool_u = torch.empty((capacity, self.d, self.H), **kw)
        self.pool_d = torch.empty((capacity, self.H, self.d), **kw)
        self.load_stream = torch.cuda.Stream(device=self.dev)
        self.slot_ready = [None] * capacity   # event: the copy into the slot finished (load stream)
        self.slot_free = [None] * capacity    # event: the last layer reading the slot finished (compute stream)
        self.bytes_loaded = 0

    def _load(self, key: int, slot: int):
        l, e = divmod(key, self.E)
        wg, wu, wd = self.layers[l]
        with torch.cuda.stream(self.load_stream):
            if self.slot_free[slot] is not None:
                self.load_stream.wait_event(self.slot_free[slot])
            self.pool_g[slot].copy_(wg[e], non_blocking=True)
            self.pool_u[slot].copy_(wu[e], non_blocking=True)
            self.pool_d[slot].copy_(wd[e], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.load_stream)
        self.slot_ready[slot] = ev
        self.bytes_loaded += 3 * self.d * self.H * 2

    def forward(self, x: torch.Tensor, logits: torch.Tensor, prefetch: bool = True):
        """x [T,H] bf16 (updated in place through all L layers), logits [T,E]. Returns (x, stats)."""
        T, H = x.shape
        E = self.E
        cache = rd.ExpertCache(self.cap, self.policy, seed=7)
        plan = rd.route(logits, 1)
        counts = plan.counts.cpu().numpy()  # the one host sync per batch: pre-gating fixes every layer
        touched = [e for e in range(E) if counts[e] > 0]
        refs = [l * E + e for l in range(self.L) for e in touched]
        cache.set_future(refs, np.arange(len(refs)))
        xs = torch.empty_like(x)
        ws = torch.empty(rd.expert_ffn_workspace_bytes(T, H, E, self.d, x.dtype), dtype=torch.uint8, device=self.dev)
        slot_tables = []
        t = 0
        comp = torch.cuda.current_stream(self.dev)

        def ensure(l):
            nonlocal t
            table = np.zeros(E, np.int32)
            for e in touched:
                hit, slot, _ev = cache.access(l * E + e, t)
                t += 1
                if not hit:
                    self._load(l * E + e, slot)
                table[e] = slot
            return table

        tables = {}
        prev_done = None
        for l in range(self.L):
            if l == 0 or not prefetch:
                if prev_done is not None:  # on demand: a layer's loads start only after the previous layer
                    self.load_stream.wait_event(prev_done)
                tables[l] = ensure(l)
            table = tables.pop(l)
            for e in touched:
                comp.wait_event(self.slot_ready[int(table[e])])
            slot_of = torch.from_numpy(table).pin_memory().to(self.dev, non_blocking=True)
            slot_tables.append(slot_of)
            rd.dispatch_rmsnorm(x, plan.dest, 1, eps=self.eps, out=xs)
            rd.expert_ffn_slots(xs, plan.offsets, slot_of, self.pool_g, self.pool_u, self.pool_d, E, src=plan.src,
                                residual=x, out=x, ws=ws)
            done = torch.cuda.Event()
            done.record(comp)
            prev_done = done
            for e in touched:
                self.slot_free[int(table[e])] = done
            if prefetch and l + 1 < self.L:
                # issued right after layer l is enqueued: copies into free slots overlap layer l's compute;
                # a copy that evicts one of layer l's slots waits for layer l (slot_free) first.
                tables[l + 1] = ensure(l + 1)
        hits, misses = cache.stats()
        return x, {"hits": hits, "misses": misses, "hit_ratio": hits / max(1, hits + misses),
                   "touched_experts": len(touched), "bytes_loaded": self.bytes_loaded}
