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
        """One batch: x [T,H] bf16 (updated in place through all L layers), logits [T,E]. Returns (x, stats)."""
        out, stats = self.run([(x, logits)], prefetch=prefetch)
        return out[0], stats

    def run(self, batches, prefetch: bool = True, policy: str | None = None):
        """Serve a queue of batches [(x, logits), ...] through the L layers. All batches are pre-gated first
        (route once each; one host read of the counts for the whole queue), so the cache knows the exact future
        reference string of (layer, expert) accesses across batches. Every layer waits only
        for its own experts; with `prefetch`, the loads of the next (batch, layer) step are issued while the
        current one computes; without it, a step's loads start after the previous step ends."""
        E = self.E
        cache = rd.ExpertCache(self.cap, policy or self.policy, seed=7)
        plans = [rd.route(lg, 1) for (_x, lg) in batches]
        counts = torch.stack([p.counts for p in plans]).cpu().numpy()
        touched = [[e for e in range(E) if c[e] > 0] for c in counts]
        steps = [(b, l) for b in range(len(batches)) for l in range(self.L)]
        refs = [l * E + e for (b, l) in steps for e in touched[b]]
        cache.set_future(refs, np.arange(len(refs)))
        comp = torch.cuda.current_stream(self.dev)
        self.slot_ready = [None] * self.cap
        self.slot_free = [None] * self.cap
        self.bytes_loaded = 0
        state = {"t": 0, "prev_first": 0}

        def ensure(step):
            """Cache decisions for one (batch, layer) step, in order. Its own experts are protected once placed;
            with prefetch the step still computing (the previous one) is protected too, so a prefetch copy never
            has to wait for that step to release a slot — unless the cache cannot hold both steps' experts, in
            which case that access falls back to protecting this step only (the copy then waits, slot_free)."""
            b, l = step
            table = np.zeros(E, np.int32)
            first = state["t"]
            guard = state["prev_first"] if prefetch else first
            for e in touched[b]:
                try:
                    hit, slot, _ev = cache.access(l * E + e, state["t"], protect_since=guard)
                except RuntimeError:
                    hit, slot, _ev = cache.access(l * E + e, state["t"], protect_since=first)
                state["t"] += 1
                if not hit:
                    self._load(l * E + e, slot)
                table[e] = slot
            state["prev_first"] = first
            return table

        work = []
        for (x, _lg), plan in zip(batches, plans):
            T, H = x.shape
            work.append((torch.empty_like(x), torch.empty(rd.expert_ffn_workspace_bytes(T, H, E, self.d, x.dtype),
                                                          dtype=torch.uint8, device=self.dev)))
        tables = {}
        prev_done = None
        for i, (b, l) in enumerate(steps):
            if i == 0 or not prefetch:
                if prev_done is not None:  # on demand: this step's loads start only after the previous step
                    self.load_stream.wait_event(prev_done)
                tables[i] = ensure((b, l))
            table = tables.pop(i)
            for e in touched[b]:
                comp.wait_event(self.slot_ready[int(table[e])])
            slot_of = torch.from_numpy(table).pin_memory().to(self.dev, non_blocking=True)
            x = batches[b][0]
            xs, ws = work[b]
            plan = plans[b]
            rd.dispatch_rmsnorm(x, plan.dest, 1, eps=self.eps, out=xs)
            rd.expert_ffn_slots(xs, plan.offsets, slot_of, self.pool_g, self.pool_u, self.pool_d, E, src=plan.src,
                                residual=x, out=x, ws=ws)
            done = torch.cuda.Event()
            done.record(comp)
            prev_done = done
            for e in touched[b]:
                self.slot_free[int(table[e])] = done
            if prefetch and i + 1 < len(steps):
                # issued right after step i is enqueued: copies into free slots overlap its compute; a copy that
                # evicts one of step i's slots waits for step i (slot_free) first.
                tables[i + 1] = ensure(steps[i + 1])
        hits, misses = cache.stats()
        return [b[0] for b in batches], {"hits": hits, "misses": misses, "hit_ratio": hits / max(1, hits + misses),
                                         "touched_experts": [len(t) for t in touched],
                                         "bytes_loaded": self.bytes_loaded}
