"""Decode serving loop with expert-aware batching (config 3; NEXT-2 of SURVEY §8(f)).

The paper's serving argument (§4.2): with pre-gating, every queued token's expert is
known before it reaches the backbone, so a batch can be formed to touch few experts; the per-token latency
of a batch grows linearly with its number of unique experts. Alg. 1 (the native
`readme_scheduler_*`, host C++) forms the batch; the baseline takes the oldest tokens first regardless of
expert (the decode-prioritized policy of §5.3). Every step runs one Llama-2-7B-shaped MoE
layer (`readme_moe_layer`) on the GPU over the scheduled tokens; time is the GPU's (CUDA events).

Synthetic workload: R requests decode concurrently; each request's next token is pre-gated with temporal
locality — it keeps the previous token's expert with probability p = 0.672 (2921/4096 tokens follow the
previous token's expert), else draws a uniform expert. A request re-enters the queue with its
next token after the step that served it.
"""
from __future__ import annotations

import numpy as np
import torch

from . import readme as rd


def simulate(policy: str, w_gate, w_up, w_down, n_requests: int = 512, max_tokens: int = 256, steps: int = 64,
             p_follow: float = 0.672, seed: int = 7, device="cuda:0", x_pool=None):
    """Run `steps` decode steps under `policy` ('expert_aware' | 'fifo'). Returns a metrics dict."""
    import synth
    E, d, H = w_gate.shape
    g = np.random.default_rng(seed)
    cur_expert = g.integers(0, E, size=n_requests).astype(np.int32)
    enq_time = np.zeros(n_requests)          # simulated time (ms) the request's current token was queued
    order = np.arange(n_requests)            # FIFO order of queued requests (fifo policy)
    sched = rd.ExpertScheduler(E) if policy == "expert_aware" else None
    if sched is not None:
        sched.push(np.arange(n_requests, dtype=np.int64), cur_expert)
    if x_pool is None:
        x_pool = synth.to_torch(synth.tokens(n_requests, H, seed=seed), "bf16").to(device)
    clock = 0.0
    uniq, lat, ms_steps, served = [], [], [], 0
    for _ in range(steps):
        if sched is not None:
            req, ex = sched.next_batch(max_tokens)
        else:
            req = order[:max_tokens].copy()
            order = order[max_tokens:]
            ex = cur_expert[req]
        B = int(req.size)
        if B == 0:
            break
        lg = torch.from_numpy(synth.logits_for_assignments(ex.astype(np.int32), E, seed=int(clock * 1000) % 100003))
        lg = lg.to(device)
        x = x_pool[torch.from_numpy(req.astype(np.int64)).to(device)]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(500_000)  # ~0.25 ms: the host enqueues the whole step first, so the events time the GPU only
        a.record()
        y, plan = rd.moe_layer(x, w_gate, w_up, w_down, k=1, logits=lg)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        clock += ms
        ms_steps.append(ms)
        uniq.append(len(np.unique(ex)))
        lat.extend((clock - enq_time[req]).tolist())
        served += B
        # the served requests decode their next token: pre-gated with temporal locality, re-queued
        follow = g.random(B) < p_follow
        nxt = np.where(follow, cur_expert[req], g.integers(0, E, size=B)).astype(np.int32)
        cur_expert[req] = nxt
        enq_time[req] = clock
        if sched is not None:
            sched.push(req.astype(np.int64), nxt)
        else:
            order = np.concatenate([order, req])
    lat = np.array(lat)
    return {"policy": policy, "steps": len(ms_steps), "tokens": served,
            "mean_unique_experts": float(np.mean(uniq)), "mean_step_ms": float(np.mean(ms_steps)),
            "tokens_per_s": served / (sum(ms_steps) * 1e-3), "mean_token_latency_ms": float(lat.mean()),
            "p95_token_latency_ms": float(np.percentile(lat, 95))}
