#!/usr/bin/env python
"""bench.py — READ-ME pre-gated MoE layer throughput on B200 (the BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl readme|reference] [--config 2]

A step is one pass of the whole hot path (route -> dispatch -> grouped gate/up GEMM
(+SiLU) -> grouped down GEMM -> combine) over one batch of synthetic tokens, through the C ABI
(libreadme_b200.so). N=1 runs BASELINE config 2 (one Llama-2-7B-shaped MoE layer, T=8192 prefill
tokens, 8 experts of d=5504 neurons, top-1, bf16). N>1 (launched by torchrun) runs the expert-parallel
layer (config 5: 65536 tokens in all, 65536/N per rank, experts sharded over ranks; all-to-alls fused into the
kernels over peer memory, with the NCCL all-to-all path timed beside it), strong scaling; value = all ranks'
tokens / max-over-ranks time.

Rank 0 prints ONE JSON line. `--impl reference` times the CPU oracle (the tier's reference arm) on a
bounded token sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer tokens/s @ Llama-2-7B shape, 1/2/4/8 B200; % bf16 TC peak / % HBM BW"
UNIT = "tokens/s"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="readme", choices=["readme", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the config-2 d=1376 / Markov / top-2 variants")
    ap.add_argument("--tokens", type=int, default=None, help="override T per rank")
    ap.add_argument("--eager", action="store_true", help="time eager calls instead of CUDA-graph replays")
    ap.add_argument("--ep", default="peer", choices=["peer", "nccl"],
                    help="N>1 expert parallelism: all-to-alls fused into the kernels over peer memory (default) "
                         "or NCCL all_to_all_single between the library's kernels")
    ap.add_argument("--no-nccl-record", action="store_true", help="N>1: skip the NCCL all-to-all sub-record")
    ap.add_argument("--offload", action="store_true",
                    help="config 4 in the memory-constrained mode (NEXT-4): experts in pinned host memory")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return FALLBACK_PEAKS, "fallback"


# ---- clocks sampler (nvidia-smi during the timed region) ----------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- L2 flush between timed steps ----------------------------------------------------------------------------

class L2Flush:
    """Between timed steps: write a 256 MiB buffer (2x L2), then read another 256 MiB, so a timed step starts
    with none of its own data in L2 AND without the flush's dirty lines, whose write-back would otherwise
    compete with the step's own DRAM stream (measured: ~126 MB of write-backs inside a decode step)."""

    NOTE = "flushed between timed steps (256 MiB written, then 256 MiB read: no step data, no dirty lines)"

    def __init__(self, dev):
        import torch
        self.w = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
        self.r = torch.zeros(64 * 1024 * 1024, dtype=torch.int32, device=dev)

    def zero_(self):
        self.w.zero_()
        self.r.sum()


# ---- workload -------------------------------------------------------------------------------------

def make_inputs(cfg: dict, T: int, rank: int, device, E_local=None, expert_base=0):
    """Synthetic Llama-2-7B-shaped inputs (recipe: DESIGN.md §Inputs). Experts are sliced on the device
    from the dense FFN by readme_build_experts (setup, untimed)."""
    import torch

    import synth
    from paper_2410_19123_b200 import readme as rd
    H, D, d, E = cfg["H"], cfg["D"], cfg["d"], cfg["E"]
    seed = synth.MASTER_SEED + 2
    wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=seed)
    S = synth.neuron_sets(E, D, d, seed=seed)
    if E_local is not None:
        S = S[expert_base:expert_base + E_local]
    dense = [synth.to_torch(w, "bf16").to(device) for w in (wg, wu, wd)]
    del wg, wu, wd
    eg, eu, ed = rd.build_experts(*dense, torch.from_numpy(np.ascontiguousarray(S)).to(device))
    dense_cpu = None
    x = synth.to_torch(synth.tokens(T, H, seed=seed + 1000 * rank), "bf16")
    lg = synth.router_logits(T, E, seed=seed + 1000 * rank)
    return dict(x=x, logits=lg, w=(eg, eu, ed), dense=dense, S=S, dense_cpu=dense_cpu)


def cpu_baseline(cfg, inp, budget_s=15.0):
    """The oracle (test infrastructure) timed on this host's cores on a bounded, expert-stratified token
    sample of the same workload; tokens are independent, so tokens/s scales linearly."""
    import oracle
    import synth
    E = cfg["E"]
    lg = inp["logits"]
    idx = lg.argmax(axis=1)
    dense = [t.cpu() for t in inp["dense"]]
    eg, eu, ed = oracle.build_experts(*dense, inp["S"])  # the oracle slices its own experts (never the GPU's)
    g = synth.rng(7, 7)
    threads = oracle.default_threads()

    def run(n_per_expert):
        sample = np.concatenate([g.choice(np.nonzero(idx == e)[0], size=n_per_expert, replace=False)
                                 for e in range(E)])
        t0 = time.perf_counter()
        yref, _ = oracle.moe_layer(inp["x"][sample], lg[sample], cfg["k"], eg, eu, ed, nthreads=threads)
        return time.perf_counter() - t0, sample, yref

    dt, s0, _ = run(4)  # calibration (32 tokens)
    per_tok = dt / s0.size
    cap = int(min(np.bincount(idx, minlength=E)))
    n_e = max(1, min(cap, int(budget_s / per_tok / E)))
    dt, sample, yref = run(n_e)
    n = sample.size
    # the oracle also on ONE thread (results are identical for any thread count), 8 tokens
    s1 = np.concatenate([g.choice(np.nonzero(idx == e)[0], size=1, replace=False) for e in range(E)])
    t0 = time.perf_counter()
    oracle.moe_layer(inp["x"][s1], lg[s1], cfg["k"], eg, eu, ed, nthreads=1)
    dt1 = time.perf_counter() - t0
    del dense
    rec = {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
           "sample": f"{n} tokens ({n_e} per expert) of config {cfg['name']}, full layer (route+dispatch+FFN+"
                     f"combine) in fp64, {dt:.1f} s",
           "single_thread": {"value": s1.size / dt1, "unit": UNIT, "sample": f"{s1.size} tokens, {dt1:.1f} s"}}
    return rec, sample, yref


def cpu_model():
    """lscpu model name of this host (the oracle's cores are named with the line)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for l in out.splitlines():
            if l.lower().startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001 - informational only
        pass
    return None


def timed_output_check(y_dev, sample, yref, dev_status):
    """The timed step's own output (the graph replays' y) on the cpu_baseline's oracle tokens, element by
    element, plus the device status word the timed steps accumulated: a number is only reported for a step
    that computed the right thing."""
    import torch
    st = int(dev_status.item())
    yg = y_dev[torch.from_numpy(sample).to(y_dev.device)].float().cpu().numpy().astype(np.float64)
    den = np.maximum(np.abs(yref).max(axis=1), 1e-6 * np.abs(yref).max())
    err = float((np.abs(yg - yref).max(axis=1) / den).max())
    ok = st == 0 and err <= 2e-2
    return {"tokens": int(sample.size), "max_rel_err": err, "tol": 2e-2, "dev_status": st, "ok": ok,
            "what": "y of the timed graph replays vs the fp64 oracle on the cpu_baseline sample tokens"}


def ep_g1_record(cfg, T, dev, args, timed):
    """Both expert-parallel paths at G = 1 (a one-rank NCCL group on this GPU, MASTER_ADDR 127.0.0.1)."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2410_19123_b200 import ep
    own = not dist.is_initialized()
    if own:
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    out = {}
    try:
        layer, lg = ep.PeerEPLayer.from_config(cfg, T, dist.group.WORLD, dev)

        def step():
            layer.route(lg)
            layer.layer(residual=True)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(args.warmup):
            g.replay()
        torch.cuda.synchronize()
        ms = float(np.mean(timed(g.replay, args.steps)))
        out["peer_memory"] = {"ms_per_step": ms, "tokens_per_s": T / (ms * 1e-3),
                              "dev_status": int(layer.dev_status.item()), "mode": "cuda_graph_replay"}
        layer.close()
        del layer
        torch.cuda.empty_cache()
        nl = ep.EPMoELayer.from_config(cfg, T, dist.group.WORLD, dev)
        for _ in range(args.warmup):
            nl.step()
        torch.cuda.synchronize()
        ms = float(np.mean(timed(nl.step, args.steps)))
        out["nccl"] = {"ms_per_step": ms, "tokens_per_s": T / (ms * 1e-3), "mode": "eager (host split sizes)"}
        del nl
        torch.cuda.empty_cache()
    finally:
        if own:
            dist.destroy_process_group()
    return out


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import synth
    world = int(os.environ.get("WORLD_SIZE", "1"))
    cfg_id = 5 if world > 1 else args.config  # the same workload as this arm's N-GPU line
    cfg = dict(synth.CONFIGS[cfg_id])
    T, H, D, d, E = cfg["T"], cfg["H"], cfg["D"], cfg["d"], cfg["E"]
    seed = synth.MASTER_SEED + 2
    wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=seed)
    S = synth.neuron_sets(E, D, d, seed=seed)
    dense = [synth.to_torch(w, "bf16") for w in (wg, wu, wd)]
    eg, eu, ed = oracle.build_experts(*dense, S)
    del wg, wu, wd
    x = synth.to_torch(synth.tokens(T, H, seed=seed), "bf16")
    lg = synth.router_logits(T, E, seed=seed)
    threads = oracle.default_threads()
    per_step = max(8, threads)  # tokens per step: a bounded sample of the workload, one per oracle thread
    g = synth.rng(5, 5)
    times = []
    for i in range(args.warmup + args.steps):
        sample = g.choice(T, size=per_step, replace=False)
        t0 = time.perf_counter()
        oracle.moe_layer(x[sample], lg[sample], cfg["k"], eg, eu, ed, nthreads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = per_step * len(times) / tot
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"config{cfg_id}_{cfg['name']}", "T": T, "H": H, "E": E, "d": d,
                       "k": cfg["k"], "tokens_per_step_sampled": per_step},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{per_step} random tokens per step of config {cfg_id}", "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _traffic(key):
    """DRAM bytes per launch of a kernel from one committed ncu --set full capture (profiles/traffic.json)."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            return json.load(f).get(key)
    return None


def run_decode(args):
    """Config 3: decode-style expert-aware batching. Per step the queued batch (B tokens with Zipf(1)-skewed
    pre-gated experts) goes through one Llama-2-7B-shaped MoE layer. HBM-bound: the
    algorithmic bytes are the weights of the experts the batch touches (U x 3*H*d*2) plus the activations.
    Also sweeps B and the number of unique experts per batch (per-token latency vs unique experts is
    linear)."""
    import torch

    import synth
    from paper_2410_19123_b200 import readme as rd
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = dict(synth.CONFIGS[3])
    H, d, E, k = cfg["H"], cfg["d"], cfg["E"], cfg["k"]
    inp = make_inputs(dict(synth.CONFIGS[2]), 512, 0, dev)
    eg, eu, ed = inp["w"]
    flush = L2Flush(dev)
    pk, pk_src = peaks()
    dev_flags = []  # dev_status of every timed decode step shape (all must be 0)

    def measure(ids):
        B = ids.shape[0]
        lg = torch.from_numpy(synth.logits_for_assignments(ids, E, seed=B)).to(dev)
        x = synth.to_torch(synth.tokens(B, H, seed=B), "bf16").to(dev)
        plan = rd.new_plan(B, E, k, dev)
        y = torch.empty_like(x)
        ws = torch.empty(rd.moe_layer_workspace_bytes(B, H, E, d, k, torch.bfloat16), dtype=torch.uint8, device=dev)
        fn = lambda: rd.moe_layer(x, eg, eu, ed, k=k, logits=lg, plan=plan, out=y, ws=ws)
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        if not args.eager:  # one CUDA graph per decode step shape (as a serving loop would)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            fn = g.replay
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
        ms = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            ms.append((a, b))
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in ms]
        U = int(len(np.unique(ids)))
        byts = U * 3.0 * H * d * 2 + 4.0 * B * H * 2
        t = float(np.mean(ms))
        st_word = int(plan.dev_status.item())
        dev_flags.append(st_word)
        if st_word:
            raise SystemExit(f"decode step B={B} set dev_status = {st_word:#x}: not reporting a number")
        return {"B": B, "unique_experts": U, "ms": t, "tokens_per_s": B / (t * 1e-3),
                "GBps": byts / (t * 1e-3) / 1e9, "hbm_frac": byts / (t * 1e-3) / 1e9 / pk["hbm_gbs"]}

    def stages(ids):
        """Live per-kernel breakdown of one decode step (per-stage graph replays, events between them, L2
        flushed): route | dispatch | expert FFN (the dominant kernel, whose roofline the line reports)."""
        B = ids.shape[0]
        lg = torch.from_numpy(synth.logits_for_assignments(ids, E, seed=B)).to(dev)
        x = synth.to_torch(synth.tokens(B, H, seed=B), "bf16").to(dev)
        plan = rd.new_plan(B, E, k, dev)
        ws_r = torch.empty(rd.route_workspace_bytes(B, E, k), dtype=torch.uint8, device=dev)
        xs = torch.empty((B * k, H), dtype=torch.bfloat16, device=dev)
        y = torch.empty_like(x)
        ws_f = torch.empty(rd.expert_ffn_workspace_bytes(B * k, H, E, d, torch.bfloat16), dtype=torch.uint8,
                           device=dev)
        fns = [lambda: rd.route(lg, k, plan=plan, ws=ws_r), lambda: rd.dispatch(x, plan.dest, k, out=xs),
               lambda: rd.expert_ffn(xs, plan.offsets, eg, eu, ed, out=y, ws=ws_f)]
        for _ in range(args.warmup):
            for f in fns:
                f()
        torch.cuda.synchronize()
        if not args.eager:
            # each stage as its own CUDA graph (as config 2 does): the events between them then time the
            # kernels, not the host-side argument marshalling and tensor-map encoding of an eager call
            graphs = []
            for f in fns:
                gph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gph):
                    f()
                graphs.append(gph)
            fns = [gph.replay for gph in graphs]
            for f in fns:
                f()
            torch.cuda.synchronize()
        rows = []
        for _ in range(args.steps):
            flush.zero_()
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(fns) + 1)]
            evs[0].record()
            for j, f in enumerate(fns):
                f()
                evs[j + 1].record()
            torch.cuda.synchronize()
            rows.append([evs[j].elapsed_time(evs[j + 1]) for j in range(len(fns))])
        return np.array(rows)

    with Clocks(0) as clk:
        sweep = [measure(synth.assignments_zipf(B, E, 1.0, seed=synth.MASTER_SEED + 3 + B))
                 for B in (64, 128, 256, 512)]
        ids256 = synth.assignments_zipf(256, E, 1.0, seed=synth.MASTER_SEED + 3 + 256)
        st = stages(ids256)
    # the Zipf exponent swept at B = 256 (s = 0 uniform, 1, 2 skewed)
    zipf = [dict(measure(synth.assignments_zipf(256, E, s_z, seed=synth.MASTER_SEED + 40 + int(s_z))), s=s_z)
            for s_z in (0.0, 1.0, 2.0)]
    uniq = [measure(synth.assignments_unique(256, u, E, seed=synth.MASTER_SEED + 30 + u)) for u in range(1, E + 1)]
    us = np.array([r["unique_experts"] for r in uniq], np.float64)
    ts = np.array([r["ms"] for r in uniq]) * 1e3
    slope, icpt = np.polyfit(us, ts, 1)
    r2 = 1 - np.sum((ts - (slope * us + icpt)) ** 2) / np.sum((ts - ts.mean()) ** 2)
    from paper_2410_19123_b200 import serving
    for pol in ("expert_aware", "fifo"):  # warm-up: first-call costs (allocations, module loads) stay out
        serving.simulate(pol, eg, eu, ed, n_requests=512, max_tokens=256, steps=8, device=dev)
    serve = [serving.simulate(pol, eg, eu, ed, n_requests=512, max_tokens=256, steps=48, device=dev)
             for pol in ("expert_aware", "fifo")]
    # the incremental router (readme_router_step) for the same 256 decode tokens: each request has a cached
    # history of 0..4095 tokens (uniform), one new token each; run once per token for the whole 32-layer model
    RW = {kk: synth.to_torch(v, "bf16").to(dev) for kk, v in synth.router_weights(n_experts=E, seed=31).items()}
    max_len = 4096
    cache = rd.new_router_cache(256, max_len, dev)
    pos = torch.from_numpy(synth.rng(32, 0).integers(0, max_len, size=256).astype(np.int32)).to(dev)
    tok = torch.from_numpy(synth.token_ids(256, seed=33)).to(dev)
    slots = torch.arange(256, dtype=torch.int32, device=dev)
    r_out = torch.empty((256, E), dtype=torch.float32, device=dev)
    r_ws = torch.empty(int(rd.lib().readme_router_step_workspace_bytes(256, max_len)), dtype=torch.uint8, device=dev)
    rstep = lambda: rd.router_step(tok, slots, pos, cache, RW, out=r_out, ws=r_ws)
    for _ in range(args.warmup):
        rstep()
    torch.cuda.synchronize()
    if not args.eager:  # a serving loop replays the step as a CUDA graph (the entry is capturable)
        r_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(r_graph):
            rstep()
        rstep = r_graph.replay
        rstep()
        torch.cuda.synchronize()
    r_ms = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rstep()
        b.record()
        torch.cuda.synchronize()
        r_ms.append(a.elapsed_time(b))
    router_ms = float(np.mean(r_ms))
    kv_bytes = float((pos.double() + 1).sum().item()) * 2 * 512 * 2
    del cache
    main_pt = sweep[2]
    U = int(len(np.unique(ids256)))
    ffn_bytes = U * 3.0 * H * d * 2 + 2.0 * 256 * k * H * 2 + 2.0 * 256 * k * d * 2  # weights + x_s, y + h
    ffn_ms = float(np.mean(st[:, 2]))
    ffn_gbs = ffn_bytes / (ffn_ms * 1e-3) / 1e9
    # e2e through the public API (readme_moe_layer) at B = 256: pinned host x/logits in, y out, every step
    x_h = synth.to_torch(synth.tokens(256, H, seed=256), "bf16").pin_memory()
    lg_h = torch.from_numpy(synth.logits_for_assignments(ids256, E, seed=256)).pin_memory()
    y_h = torch.empty_like(x_h).pin_memory()
    x_d, lg_d = torch.empty_like(x_h, device=dev), torch.empty_like(lg_h, device=dev)
    y_d = torch.empty_like(x_d)
    plan_e = rd.new_plan(256, E, k, dev)
    ws_e = torch.empty(rd.moe_layer_workspace_bytes(256, H, E, d, k, torch.bfloat16), dtype=torch.uint8, device=dev)

    def e2e_step():
        x_d.copy_(x_h, non_blocking=True)
        lg_d.copy_(lg_h, non_blocking=True)
        rd.moe_layer(x_d, eg, eu, ed, k=k, logits=lg_d, plan=plan_e, out=y_d, ws=ws_e)
        y_h.copy_(y_d, non_blocking=True)

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        e2e_step()
        b.record()
        torch.cuda.synchronize()
        e_ms.append(a.elapsed_time(b))
    # the same batches streamed through HostPipeline (H2D of batch i+1 and D2H of batch i-1 overlap the layer of
    # batch i; every batch's bytes still cross PCIe)
    from paper_2410_19123_b200.pipeline import HostPipeline
    pipe = HostPipeline(256, H, E, k, eg, eu, ed, device=dev)
    ys_h = [torch.empty_like(x_h).pin_memory() for _ in range(2)]
    nb = max(8, args.steps)
    pipe.run([x_h] * 2, [lg_h] * 2, ys_h)
    torch.cuda.synchronize()
    pa = torch.cuda.Event(enable_timing=True)
    pa.record(pipe.up)
    last = pipe.run([x_h] * nb, [lg_h] * nb, [ys_h[i % 2] for i in range(nb)])
    pb = torch.cuda.Event(enable_timing=True)
    for ev in last:
        if ev is not None:
            pipe.down.wait_event(ev)
    pb.record(pipe.down)
    torch.cuda.synchronize()
    p_ms = pa.elapsed_time(pb) / nb
    line = {"metric": METRIC, "value": main_pt["tokens_per_s"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main_pt["ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "config3_decode_batching", "B": 256, "H": H, "D": cfg["D"], "E": E, "d": d,
                       "k": k, "assignments": "Zipf(s=1) over experts", "l2": L2Flush.NOTE},
            "dev_status": max(dev_flags) if dev_flags else 0,
            "roofline": {"bound": "hbm", "kernel": "expert FFN (ffn_layer2_kernel, one launch per step)",
                         "achieved": ffn_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ffn_gbs / pk["hbm_gbs"],
                         "traffic": _traffic("decode_expert_ffn_bytes_per_launch"),
                         "algorithmic": f"U*3*H*d*2 (touched experts' weights) + 2*B*H*2 + 2*B*d*2 = "
                                        f"{ffn_bytes:.4g} B per launch (U={U})",
                         "peak_source": f"{pk_src} HBM copy (MEASURED_PEAKS.json)",
                         "step_GBps": main_pt["GBps"], "step_frac": main_pt["hbm_frac"]},
            "stage_ms_mean": {"route": float(np.mean(st[:, 0])), "dispatch": float(np.mean(st[:, 1])),
                              "expert_ffn": ffn_ms},
            "router_step": {"ms": router_ms, "kv_GBps": kv_bytes / (router_ms * 1e-3) / 1e9,
                            "share_of_32_layer_step": router_ms / (router_ms + 32 * main_pt["ms"]),
                            "note": "readme_router_step: 256 decode tokens, cached histories uniform in [0, 4096), "
                                    "once per token for all 32 layers; paper: router 1.26-1.50 % of batched step "
                                    "latency (PAPER.md:647)"},
            "e2e": {"value": 256 / (p_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": x_h.numel() * 2 + lg_h.numel() * 4, "d2h_bytes_per_step": y_h.numel() * 2,
                    "ms_per_step": p_ms,
                    "mode": "pipelined over K batches (HostPipeline: H2D / layer / D2H on three streams)",
                    "serial": {"value": 256 / (float(np.mean(e_ms)) * 1e-3), "ms_per_step": float(np.mean(e_ms)),
                               "note": "one batch at a time: H2D, layer, D2H back to back"}},
            "clocks": clk.summary(),
            "decode_sweep": sweep,
            "zipf_sweep": zipf,
            "unique_expert_sweep": {"points": uniq, "us_per_extra_expert": float(slope), "intercept_us": float(icpt),
                                    "r2_linear": float(r2), "paper": "linear per-token latency in unique experts "
                                                                   "(PAPER.md:234, fig:batching b)"},
            "serving_sim": {"runs": serve, "paper": "mean unique experts per batch 3.51 (READ-ME) vs 5.08 / 5.21 "
                                                   "(decode- / prefill-prioritized), PAPER.md:426; A100 trace replay",
                            "workload": "512 concurrent requests, MaxTokenLen 256, locality p=0.672, 48 steps, "
                                        "one Llama-2-7B-shape MoE layer per step on the GPU"},
            "gpu_launches": 3 * args.steps}  # route (one cluster launch), dispatch, expert FFN
    print(json.dumps(line), flush=True)


def run_tiny(args):
    """Config 1: the tiny fp32 layer (E=8, top-1, H=64, expert width 128, T=256) — latency only (SURVEY
    §8(d)); the CUDA-core fp32 path (no TF32)."""
    import torch

    import synth
    from paper_2410_19123_b200 import readme as rd
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    c = synth.CONFIGS[1]
    T, H, d, E, k = c["T"], c["H"], c["d"], c["E"], c["k"]
    seed = synth.MASTER_SEED + 1
    x = synth.to_torch(synth.tokens(T, H, seed=seed), "f32").to(dev)
    lg = torch.from_numpy(synth.router_logits(T, E, seed=seed)).to(dev)
    W = [synth.to_torch(w, "f32").to(dev) for w in synth.expert_weights(E, d, H, seed=seed)]
    plan = rd.new_plan(T, E, k, dev)
    y = torch.empty_like(x)
    ws = torch.empty(rd.moe_layer_workspace_bytes(T, H, E, d, k, torch.float32), dtype=torch.uint8, device=dev)
    fn = lambda: rd.moe_layer(x, *W, k=k, logits=lg, plan=plan, out=y, ws=ws)
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    flush = L2Flush(dev)
    ms = []
    with Clocks(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            ms.append((a, b))
        torch.cuda.synchronize()
    t = float(np.mean([a.elapsed_time(b) for a, b in ms]))
    line = {"metric": METRIC, "value": T / (t * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config1_tiny", "T": T, "H": H, "E": E, "d": d, "k": k,
                       "note": "latency-bound (12.6 MFLOP); graph replay", "l2": L2Flush.NOTE},
            "latency_us": t * 1e3, "gpu_launches": 2 * args.steps,  # route, one-launch fp32 FFN (a5 gather + a6 + a7 + a8)
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def run_stack(args):
    """Config 4: the full 32-layer refactored MoE stack (MoE-only pre-norm, reading Q10), T = 16384 tokens
    (4 requests x 4096, Markov expert locality p = 0.672), routed ONCE per request batch
     — one readme_moe_stack call per step."""
    import torch

    import synth
    from paper_2410_19123_b200 import readme as rd
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = dict(synth.CONFIGS[4])
    T, H, d, E, k, L = args.tokens or cfg["T"], cfg["H"], cfg["d"], cfg["E"], cfg["k"], cfg["L"]
    seed = synth.MASTER_SEED + 4
    layers = [synth.expert_weights_device(E, d, H, dev, seed=seed, layer=l) for l in range(L)]
    ids = synth.assignments_markov(T // 4096 if T >= 4096 else 1, min(T, 4096), E, 0.672, seed=seed)
    lg = torch.from_numpy(synth.logits_for_assignments(ids, E, seed=seed)).to(dev)
    x0 = synth.to_torch(synth.tokens(T, H, seed=seed), "bf16").to(dev)
    x = torch.empty_like(x0)
    plan = rd.new_plan(T, E, k, dev)
    ws = torch.empty(rd.moe_stack_workspace_bytes(T, H, E, d, k, torch.bfloat16), dtype=torch.uint8, device=dev)
    flush = L2Flush(dev)

    def step():
        x.copy_(x0)
        rd.moe_stack(x, layers, k=k, logits=lg, plan=plan, ws=ws)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ms = []
    with Clocks(0) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            ms.append((a, b))
        torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ms]
    t = float(np.mean(ms))
    # the pre-gating router G (one causal block + gating head) over the same requests, once per step
    RW = {kk: synth.to_torch(v, "bf16").to(dev) for kk, v in synth.router_weights(n_experts=E, seed=seed).items()}
    ids = torch.from_numpy(synth.token_ids(T, seed=seed)).to(dev)
    starts = torch.arange(0, T + 1, min(T, 4096), dtype=torch.int32, device=dev)
    r_ws = torch.empty(rd.router_workspace_bytes(T, starts.numel() - 1), dtype=torch.uint8, device=dev)
    r_out = torch.empty((T, E), dtype=torch.float32, device=dev)
    rfn = lambda: rd.router_forward(ids, starts, RW, out=r_out, ws=r_ws)
    for _ in range(args.warmup):
        rfn()
    torch.cuda.synchronize()
    rms = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rfn()
        b.record()
        rms.append((a, b))
    torch.cuda.synchronize()
    router_ms = float(np.mean([a.elapsed_time(b) for a, b in rms]))
    e2e = None
    if not args.no_e2e:
        # e2e through the public API: the step's tokens and logits from pinned host memory, the 32-layer
        # stack, the result back to pinned host memory — one batch at a time (the PCIe copies are ~5 % of a
        # ~60 ms step, so no pipelining)
        x_h = x0.cpu().pin_memory()
        lg_h = lg.cpu().pin_memory()
        y_h = torch.empty_like(x_h).pin_memory()
        lg_d = torch.empty_like(lg)

        def e2e_step():
            x.copy_(x_h, non_blocking=True)
            lg_d.copy_(lg_h, non_blocking=True)
            rd.moe_stack(x, layers, k=k, logits=lg_d, plan=plan, ws=ws)
            y_h.copy_(x, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        ems = []
        for _ in range(max(2, args.steps)):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            e2e_step()
            b.record()
            ems.append((a, b))
        torch.cuda.synchronize()
        e_ms = float(np.mean([a.elapsed_time(b) for a, b in ems]))
        e2e = {"value": T / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": x_h.numel() * 2 + lg_h.numel() * 4,
               "d2h_bytes_per_step": y_h.numel() * 2, "ms_per_step": e_ms,
               "mode": "one batch at a time: H2D, 32-layer stack, D2H"}
    pk, pk_src = peaks()
    flops = L * 6.0 * T * k * H * d
    ach = flops / (t * 1e-3) / 1e12
    peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    line = {"metric": METRIC, "value": T / (t * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "config4_stack32", "T": T, "L": L, "H": H, "E": E, "d": d, "k": k,
                       "routing": "Markov locality p=0.672, routed once per step", "l2": L2Flush.NOTE},
            "layer_tokens_per_s": T * L / (t * 1e-3),
            "router": {"ms": router_ms, "share_of_step_with_router": router_ms / (router_ms + t),
                       "note": "readme_router_forward over the same T tokens (4096-token sequences), run once per "
                               "request, not per layer; paper: AR router 1.26-1.50 % of step latency (PAPER.md:647)"},
            "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                         "traffic": None, "algorithmic": f"L*6*T*k*H*d = {flops:.4g} FLOP per step",
                         "peak_source": f"{pk_src} bf16 sustained (kernels timed inside a ~60 ms step)",
                         "frac_of_burst": ach / pk["bf16_tflops"]},
            "dev_status": int(plan.dev_status.item()),
            "gpu_launches": (1 + 2 * L) * args.steps, "clocks": clk.summary()}  # route, L x (norm-dispatch, FFN)
    if e2e is not None:
        line["e2e"] = e2e
    print(json.dumps(line), flush=True)


def run_offload(args):
    """Config 4, memory-constrained mode (NEXT-4 of SURVEY §8(f)): the experts of
    L layers live in pinned host memory and only `cap` expert slots fit on the device. A queue of Q pre-gated
    batches (T tokens each, u experts per batch as expert-aware batching yields them) runs through the L
    layers; the makespan of the queue is timed with CUDA events for fine-grained prefetching (next step's
    experts load on a separate stream while this step computes) vs on-demand loading, under the
    Belady-inspired and LRU caches. (The paper's cache-hit table, tab:cache-hit, needs its Chatbot-Arena trace:
    out of scope.)"""
    import torch

    import synth
    from paper_2410_19123_b200 import readme as rd
    from paper_2410_19123_b200.offload import OffloadedStack
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = dict(synth.CONFIGS[4])
    H, d, E = cfg["H"], cfg["d"], cfg["E"]
    L, Q, u = 8, 8, 2
    T = args.tokens or 8192
    seed = synth.MASTER_SEED + 40
    host = []
    for l in range(L):
        ws = synth.expert_weights_device(E, d, H, dev, seed=seed, layer=l)
        host.append(tuple(w.cpu().pin_memory() for w in ws))
        del ws
    torch.cuda.empty_cache()
    x0s, lgs, touched = [], [], []
    for b in range(Q):
        ids = synth.assignments_unique(T, u, E, seed=seed + 100 + b)
        lgs.append(torch.from_numpy(synth.logits_for_assignments(ids, E, seed=seed + 200 + b)).to(dev))
        x0s.append(synth.to_torch(synth.tokens(T, H, seed=seed + 300 + b), "bf16").to(dev))
        touched.append(sorted(set(ids.tolist())))
    flush = L2Flush(dev)
    expert_bytes = 3 * d * H * 2
    runs = []
    with Clocks(0) as clk:
        for cap in (4, 8, 16):
            for policy in ("belady", "lru"):
                st = OffloadedStack(host, cap, policy, dev)
                for prefetch in (True, False):
                    ms = []
                    for it in range(args.warmup + args.steps):
                        batches = [(x.clone(), lg) for x, lg in zip(x0s, lgs)]
                        flush.zero_()
                        torch.cuda.synchronize()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record()
                        _, stats = st.run(batches, prefetch=prefetch)
                        b.record()
                        torch.cuda.synchronize()
                        if it >= args.warmup:
                            ms.append(a.elapsed_time(b))
                    t = float(np.mean(ms))
                    runs.append({"cap_slots": cap, "policy": policy, "prefetch": prefetch, "ms": t,
                                 "tokens_per_s": Q * T / (t * 1e-3), "hit_ratio": stats["hit_ratio"],
                                 "misses": stats["misses"], "h2d_GBps": stats["bytes_loaded"] / (t * 1e-3) / 1e9})
                del st
                torch.cuda.empty_cache()
    for r in runs:
        if r["prefetch"]:
            od = next(q for q in runs if q["cap_slots"] == r["cap_slots"] and q["policy"] == r["policy"]
                      and not q["prefetch"])
            r["latency_reduction_vs_on_demand"] = 1.0 - r["ms"] / od["ms"]
    # the same Q batches with all L*E experts resident (readme_moe_stack per batch): the floor
    dev_layers = [tuple(w.to(dev) for w in ly) for ly in host]
    res_ms = []
    for it in range(args.warmup + args.steps):
        xs = [x.clone() for x in x0s]
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for xb, lg in zip(xs, lgs):
            rd.moe_stack(xb, dev_layers, logits=lg)
        b.record()
        torch.cuda.synchronize()
        if it >= args.warmup:
            res_ms.append(a.elapsed_time(b))
    resident_ms = float(np.mean(res_ms))
    del dev_layers
    # H2D copy bandwidth of one expert from pinned memory (the load stream's roofline)
    src = torch.cat([w[0].reshape(-1) for w in host[0]]).pin_memory()
    slot = torch.empty_like(src, device=dev)
    h2d = []
    for it in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        slot.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            h2d.append(a.elapsed_time(b))
    h2d_GBps = expert_bytes / (float(np.median(h2d)) * 1e-3) / 1e9
    best = max((r for r in runs if r["prefetch"]), key=lambda r: r["tokens_per_s"])
    line = {"metric": "memory-constrained MoE stack tokens/s (experts in host memory, NEXT-4)",
            "value": best["tokens_per_s"], "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": best["ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "config4_offload", "Q_batches": Q, "T": T, "L": L, "H": H, "E": E, "d": d,
                       "experts_per_batch": u, "host_expert_bytes": L * E * expert_bytes,
                       "routing": "expert-aware batches (u experts each), routed once per batch",
                       "l2": L2Flush.NOTE},
            "runs": runs, "resident_ms": resident_ms, "h2d_expert_GBps": h2d_GBps,
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == 3 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        run_decode(args)
        return
    if args.config == 1 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        run_tiny(args)
        return
    if args.config == 4 and args.offload and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        run_offload(args)
        return
    if args.config == 4 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        run_stack(args)
        return
    import torch
    import torch.distributed as dist

    import synth
    from paper_2410_19123_b200 import readme as rd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # README_BENCH_BACKEND=gloo lets several ranks share one GPU (a functional check of the N>1 path only:
        # their kernels time-slice, so the numbers mean nothing)
        backend = os.environ.get("README_BENCH_BACKEND", "nccl")
        if backend != "nccl":
            local = local % torch.cuda.device_count()
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)} if backend == "nccl" else {}))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = dict(synth.CONFIGS[args.config if world == 1 else 5])
    # N > 1: config 5 as BASELINE.json states it, 65536 tokens in all, strong scaling (65536 / N per rank)
    T = args.tokens or (cfg["T"] if world == 1 else cfg["T"] // world)
    H, d, E, k = cfg["H"], cfg["d"], cfg["E"], cfg["k"]

    flush = L2Flush(dev)

    def timed(fn, n):
        """n steps, L2 flushed before each (outside the events), CUDA events on the launching stream."""
        out = []
        for _ in range(n):
            flush.zero_()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            fn()
            s1.record()
            out.append((s0, s1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in out]

    ep_mode, ep_fallback = args.ep, None
    if world > 1:
        from paper_2410_19123_b200 import ep
        layer = None
        if ep_mode == "peer":
            # peer-memory EP needs CUDA IPC mappings between the ranks' GPUs; if any rank cannot set them up,
            # every rank falls back to the NCCL all-to-all path (decided collectively, reported in the line)
            try:
                layer, lg_ep = ep.PeerEPLayer.from_config(cfg, T, dist.group.WORLD, dev)
                ok = 1
            except Exception as e:  # noqa: BLE001 - any setup failure selects the fallback
                ok, ep_fallback = 0, f"peer-memory setup failed on rank {rank}: {type(e).__name__}: {e}"[:300]
            flag = torch.tensor([ok], device=dev, dtype=torch.int32)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                if layer is not None:
                    layer.close()
                ep_mode = "nccl"
                ep_fallback = ep_fallback or "peer-memory setup failed on another rank"
        if ep_mode == "peer":
            def step_fn():  # route once (+ count exchange on the device), then the fused layer
                layer.route(lg_ep)
                layer.layer(residual=True)
        else:
            layer = ep.EPMoELayer.from_config(cfg, T, dist.group.WORLD, dev)
            step_fn = layer.step
    else:
        inp = make_inputs(cfg, T, rank, dev)
        eg, eu, ed = inp["w"]
        x_dev = inp["x"].to(dev)
        lg_dev = torch.from_numpy(inp["logits"]).to(dev)
        plan = rd.new_plan(T, E, k, dev)
        y = torch.empty_like(x_dev)
        ws = torch.empty(rd.moe_layer_workspace_bytes(T, H, E, d, k, torch.bfloat16), dtype=torch.uint8, device=dev)

        def step_fn():  # the whole hot path through the public C entry (route + fused grouped GEMMs)
            rd.moe_layer(x_dev, eg, eu, ed, k=k, logits=lg_dev, plan=plan, out=y, ws=ws)

    for _ in range(args.warmup):
        step_fn()
    torch.cuda.synchronize()
    if world > 1 and ep_mode == "peer":
        # a peer-memory exchange that never completes makes readme_ep_wait flag README_DEV_EP_TIMEOUT after
        # ~10 s instead of hanging; if any rank saw that during warm-up, every rank switches to NCCL
        bad = torch.tensor([int(layer.dev_status.item()) & rd.README_DEV_EP_TIMEOUT], device=dev, dtype=torch.int32)
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if int(bad.item()):
            layer.close()
            ep_mode, ep_fallback = "nccl", "peer-memory exchange timed out during warm-up (README_DEV_EP_TIMEOUT)"
            layer = ep.EPMoELayer.from_config(cfg, T, dist.group.WORLD, dev)
            step_fn = layer.step
            for _ in range(args.warmup):
                step_fn()
            torch.cuda.synchronize()
    eager_fn = step_fn
    if (world == 1 or ep_mode == "peer") and not args.eager:
        # The C ABI is stream-ordered and allocation-free, so the whole step captures into one CUDA graph
        # (how a fixed-shape serving step runs); replays remove the per-call host launch cost.
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step_fn()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_fn()
        step_fn = graph.replay
        for _ in range(args.warmup):
            step_fn()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if world == 1:
        ws_r = torch.empty(rd.route_workspace_bytes(T, E, k), dtype=torch.uint8, device=dev)
        xs = torch.empty((T * k, H), dtype=torch.bfloat16, device=dev)
        hbuf = torch.empty((T * k, d), dtype=torch.bfloat16, device=dev)
        y2 = torch.empty_like(x_dev)
        ws_f = torch.empty(rd.expert_ffn_workspace_bytes(T * k, H, E, d, torch.bfloat16), dtype=torch.uint8,
                           device=dev)
        stage_fns = [lambda: rd.route(lg_dev, k, plan=plan, ws=ws_r),
                     lambda: rd.dispatch(x_dev, plan.dest, k, out=xs),
                     lambda: rd.expert_ffn(xs, plan.offsets, eg, eu, ed, out=y2, ws=ws_f)]
        # each stage as its own CUDA graph: replays launch with ~us of host work, so the events between them
        # measure the kernels rather than the Python/ctypes/tensor-map set-up of an eager call
        stage_graphs = []
        for f in stage_fns:
            f()
            torch.cuda.synchronize()
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                f()
            stage_graphs.append(gph)
        stage_fns = [gph.replay for gph in stage_graphs]
    with Clocks(local) as clk:
        if world > 1:
            step_ms = timed(step_fn, args.steps)
        else:
            # K timed steps (graph replays of readme_moe_layer); after each, in the same thermal/power
            # window, one pass through the per-row C entries (each a graph replay) with events between them
            # gives the live per-kernel breakdown (route | dispatch | expert FFN).
            step_ms, eager_ms, stages = [], [], []
            for _ in range(args.steps):
                step_ms += timed(step_fn, 1)
                eager_ms += timed(eager_fn, 1)
                flush.zero_()
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(stage_fns) + 1)]
                evs[0].record()
                for j, f in enumerate(stage_fns):
                    f()
                    evs[j + 1].record()
                torch.cuda.synchronize()
                stages.append([evs[j].elapsed_time(evs[j + 1]) for j in range(len(stage_fns))])
            st = np.array(stages)
            route_ms, disp_ms, ffn_ms = (st[:, j] for j in range(3))
            # the two projections as separate launches (readme_expert_gate_up / _down), for reference
            gu_ms = timed(lambda: rd.expert_gate_up(xs, plan.offsets, eg, eu, out=hbuf), max(3, args.steps // 3))
            dn_ms = timed(lambda: rd.expert_down(hbuf, plan.offsets, ed, src=plan.src, out=y2), max(3, args.steps // 3))
    if world > 1:
        dist.barrier()
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = T * world / (ms_per_step * 1e-3)

    pk, pk_src = peaks()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": (f"config{args.config}_{cfg['name']}" if world == 1 else "config5_expert_parallel"),
                       "T_per_gpu": T, "T_total": T * world, "H": H, "D": cfg["D"], "E": E, "d": d, "k": k,
                       "parallelism": "single" if world == 1 else f"ep{world}",
                       **({} if world == 1 else {"ep_exchange": "peer-memory stores fused into the dispatch kernel "
                                                 "and the down-GEMM epilogue" if ep_mode == "peer" else
                                                 "NCCL all_to_all_single"}),
                       **({"ep_fallback": ep_fallback} if ep_fallback else {}),
                       "l2": L2Flush.NOTE}}
    if world == 1:
        med = lambda a: float(np.median(a))
        line["step_mode"] = "cuda_graph_replay" if not args.eager else "eager"
        line["eager_ms_per_step"] = float(np.mean(eager_ms))
        # SURVEY §8(d) protocol extras: spread of the timed (cold-L2) steps, and warm steps back to back
        line["ms_p10_p50_p90"] = [float(np.percentile(step_ms, q)) for q in (10, 50, 90)]
        warm = []
        wa = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        wa[0].record()
        for j in range(args.steps):
            step_fn()
            wa[j + 1].record()
        torch.cuda.synchronize()
        warm = [wa[j].elapsed_time(wa[j + 1]) for j in range(args.steps)]
        line["warm_ms_per_step"] = float(np.mean(warm))
        line["stage_ms_median"] = {"step": med(step_ms), "route": med(route_ms), "dispatch": med(disp_ms),
                                   "expert_ffn": med(ffn_ms)}
        f_all, f_gu, f_dn = 6.0 * T * k * H * d, 4.0 * T * k * H * d, 2.0 * T * k * H * d
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get("expert_ffn_bytes_per_launch")
        ach = f_all / (float(np.mean(ffn_ms)) * 1e-3) / 1e12
        a_gu = f_gu / (float(np.mean(gu_ms)) * 1e-3) / 1e12
        a_dn = f_dn / (float(np.mean(dn_ms)) * 1e-3) / 1e12
        # the roofline is the measured bf16 BURST peak (cuBLAS timed alone, like this launch); the sustained
        # (power-capped, back-to-back for seconds) figure is reported beside it, never instead of it
        peak = pk["bf16_tflops"]
        peak_sus = pk.get("bf16_tflops_sustained")
        if T != 8192:
            traffic = None  # the committed capture is of config 2 (T = 8192)
        line["roofline"] = {"bound": "tensor",
                            "kernel": "grouped expert FFN: a6 gate/up GEMM + SiLU*up and a7 down GEMM in ONE persistent "
                                      "tcgen05 cta_group::2 launch (ffn_layer2_kernel) = readme_expert_ffn",
                            "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                            "frac": ach / peak, "traffic": traffic,
                            "peak_source": f"{pk_src} bf16 burst (MEASURED_PEAKS.json)",
                            "frac_of_sustained": (ach / peak_sus) if peak_sus else None,
                            "algorithmic": f"6*T*k*H*d = {f_all:.4g} FLOP per launch",
                            "split_launches": {"gate_up_tflops": a_gu, "gate_up_frac": a_gu / peak,
                                               "down_combine_tflops": a_dn, "down_combine_frac": a_dn / peak}}
        # the standalone permutation entries (readme_dispatch / readme_combine), HBM-bound. Each is captured
        # in a CUDA graph and replayed (an eager launch's host gap would land inside its events), L2 flushed.
        ys = torch.empty_like(xs)

        def graph_of(fn):
            fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            return g.replay

        # measured on 8x the rows (65536 tokens, 512 MiB each way) so the ~5 us launch of a one-kernel
        # graph does not dominate a 20 us kernel; same kernels, same per-row work
        Tb = 8 * T
        xb = x_dev.repeat(8, 1)
        lgb = torch.from_numpy(synth.router_logits(Tb, E, seed=synth.MASTER_SEED + 77)).to(dev)
        planb = rd.route(lgb, k)
        xsb = torch.empty((Tb * k, H), dtype=torch.bfloat16, device=dev)
        ysb = torch.empty_like(xsb)
        yb = torch.empty_like(xb)
        disp_g_ms = timed(graph_of(lambda: rd.dispatch(xb, planb.dest, k, out=xsb)), args.steps)
        comb_ms = timed(graph_of(lambda: rd.combine(ysb, planb.dest, planb.topk_w, k, out=yb)), args.steps)
        del xb, xsb, ysb, yb
        hbm = pk["hbm_gbs"]
        disp_bytes = 2.0 * Tb * k * H * 2
        comb_bytes = (k + 1.0) * Tb * H * 2
        dg = disp_bytes / (med(disp_g_ms) * 1e-3) / 1e9
        cg = comb_bytes / (med(comb_ms) * 1e-3) / 1e9
        line["hbm"] = {"dispatch_GBps": dg, "combine_GBps": cg, "peak_GBps": hbm, "dispatch_frac": dg / hbm,
                       "combine_frac": cg / hbm, "rows": Tb * k,
                       "note": "standalone entries readme_dispatch (scatter) and readme_combine (k=1 gather), "
                               "both bulk-copy row moves at this size; inside readme_moe_layer the dispatch is the "
                               "gather form overlapped with the FFN and the k=1 combine is fused into the down GEMM "
                               "epilogue; graph-replayed at 8x config-2 rows, L2 flushed"}
        line["gpu_launches"] = (3 if k == 1 else 4) * args.steps  # route + dispatch + expert FFN (+combine)
    else:
        # peer: route, publish, (signal, wait) x3, plan, dispatch, FFN = 11; nccl: route, dispatch, FFN,
        # combine (+ NCCL's own kernels)
        line["gpu_launches"] = (11 if ep_mode == "peer" else 4) * args.steps
        line["step_mode"] = "cuda_graph_replay" if (ep_mode == "peer" and not args.eager) else "eager"
        # whole-step tensor roofline per rank: the rank's expert FFN FLOPs (its experts' rows: T per rank on
        # average) over the max-over-ranks step time, which also holds the exchange phases
        f_rank = 6.0 * T * k * H * d
        ach = f_rank / (ms_per_step * 1e-3) / 1e12
        line["roofline"] = {"bound": "tensor", "kernel": "whole expert-parallel step per rank (dispatch with the "
                            "all-to-all, grouped expert FFN with the return all-to-all, flag phases)",
                            "achieved": ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                            "frac": ach / pk["bf16_tflops"], "traffic": None,
                            "algorithmic": f"6*T_rank*k*H*d = {f_rank:.4g} FLOP per rank per step",
                            "peak_source": f"{pk_src} bf16 burst (MEASURED_PEAKS.json)"}
    line["clocks"] = clk.summary()

    if world == 1 and args.config == 5 and not args.no_variants:
        # config 5's expert-parallel machinery at G = 1 on this GPU (a one-rank process group): the fused
        # peer-memory step (route + count publish + plan, dispatch with the all-to-all stores, the FFN whose down
        # epilogue returns rows, three flag phases) and the NCCL all-to-all step, on the same 65536 tokens —
        # the per-step cost of the EP machinery beside the plain layer above
        line["ep_g1"] = ep_g1_record(cfg, T, dev, args, timed)

    if world == 1 and args.config == 2 and not args.no_variants:
        # SURVEY §8(d) config-2 variants: the d = D/8 = 1376 partition experts, Markov-locality routing
        # (2 requests x 4096, p = 0.672), and top-2. Each: graph-replayed readme_moe_layer step and the
        # expert-FFN launch alone (events, L2 flushed), same protocol as the main line.
        def variant(name, d_v, k_v, lg_np, w_v):
            eg_v, eu_v, ed_v = w_v
            lg_v = torch.from_numpy(lg_np).to(dev)
            plan_v = rd.new_plan(T, E, k_v, dev)
            y_v = torch.empty_like(x_dev)
            ws_v = torch.empty(rd.moe_layer_workspace_bytes(T, H, E, d_v, k_v, torch.bfloat16), dtype=torch.uint8,
                               device=dev)
            fn = lambda: rd.moe_layer(x_dev, eg_v, eu_v, ed_v, k=k_v, logits=lg_v, plan=plan_v, out=y_v, ws=ws_v)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            st_ms = timed(g.replay, args.steps)
            xs_v = torch.empty((T * k_v, H), dtype=torch.bfloat16, device=dev)
            rd.dispatch(x_dev, plan_v.dest, k_v, out=xs_v)
            ys_v = torch.empty_like(xs_v)
            wsf = torch.empty(rd.expert_ffn_workspace_bytes(T * k_v, H, E, d_v, torch.bfloat16), dtype=torch.uint8,
                              device=dev)
            f_ms = timed(lambda: rd.expert_ffn(xs_v, plan_v.offsets, eg_v, eu_v, ed_v, out=ys_v, ws=wsf), args.steps)
            tf = 6.0 * T * k_v * H * d_v / (float(np.mean(f_ms)) * 1e-3) / 1e12
            return {"variant": name, "d": d_v, "k": k_v, "tokens_per_s": T / (float(np.mean(st_ms)) * 1e-3),
                    "ms_per_step": float(np.mean(st_ms)), "expert_ffn_ms": float(np.mean(f_ms)),
                    "expert_ffn_tflops": tf, "frac": tf / pk["bf16_tflops"],
                    "max_expert_rows": int(plan_v.counts.max().item())}
        seedv = synth.MASTER_SEED + 22
        variants = [
            variant("d1376_partition", 1376, 1, inp["logits"],
                    synth.expert_weights_device(E, 1376, H, dev, seed=seedv)),
            variant("markov_locality_2x4096", d, 1,
                    synth.logits_for_assignments(synth.assignments_markov(2, T // 2, E, 0.672, seed=seedv), E,
                                                 seed=seedv), (eg, eu, ed)),
            variant("top2", d, 2, inp["logits"], (eg, eu, ed)),
        ]
        line["variants"] = variants

    if world == 1 and not args.no_e2e:
        # e2e through the public API (readme_moe_layer) with pinned host buffers: H2D inputs, D2H result.
        x_h = inp["x"].pin_memory()
        lg_h = torch.from_numpy(inp["logits"]).pin_memory()
        y_h = torch.empty_like(x_h).pin_memory()
        x_d = torch.empty_like(x_dev)
        lg_d = torch.empty_like(lg_dev)
        y_d = torch.empty_like(x_dev)

        def e2e_step():
            x_d.copy_(x_h, non_blocking=True)
            lg_d.copy_(lg_h, non_blocking=True)
            rd.moe_layer(x_d, eg, eu, ed, k=k, logits=lg_d, plan=plan, out=y_d, ws=ws)
            y_h.copy_(y_d, non_blocking=True)

        for _ in range(max(2, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        e_ms = timed(e2e_step, args.steps)
        serial = {"value": T / (np.mean(e_ms) * 1e-3), "ms_per_step": float(np.mean(e_ms)),
                  "note": "one batch at a time: H2D, layer, D2H back to back"}
        # the same K batches streamed through paper_2410_19123_b200.pipeline.HostPipeline: uploads of batch
        # i+1 and downloads of batch i-1 overlap the layer of batch i (every batch's bytes still cross PCIe)
        from paper_2410_19123_b200.pipeline import HostPipeline
        pipe = HostPipeline(T, H, E, k, eg, eu, ed, device=dev)
        xs_h = [x_h] * args.steps
        lgs_h = [lg_h] * args.steps
        ys_h = [torch.empty_like(x_h).pin_memory() for _ in range(2)]
        pipe.run(xs_h[:2], lgs_h[:2], ys_h)
        torch.cuda.synchronize()
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        a.record(pipe.up)
        last = pipe.run(xs_h, lgs_h, [ys_h[i % 2] for i in range(args.steps)])
        bevt = torch.cuda.Event(enable_timing=True)
        for ev in last:
            if ev is not None:
                pipe.down.wait_event(ev)
        bevt.record(pipe.down)
        torch.cuda.synchronize()
        p_ms = a.elapsed_time(bevt) / args.steps
        line["e2e"] = {"value": T / (p_ms * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": x_h.numel() * 2 + lg_h.numel() * 4,
                       "d2h_bytes_per_step": y_h.numel() * 2, "ms_per_step": p_ms,
                       "mode": "pipelined over K batches (HostPipeline: H2D / layer / D2H on three streams)",
                       "serial": serial}
        # the e2e roofline: this step's bytes copied both ways at once on the copy streams, no compute
        xd2 = torch.empty_like(x_d)

        def copies_only():
            # the copy streams start after the timing event on the current stream (without these waits they
            # would begin during timed()'s L2 flush, before the start event, and the time would read short)
            pipe.up.wait_stream(torch.cuda.current_stream())
            pipe.down.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(pipe.up):
                xd2.copy_(x_h, non_blocking=True)
                lg_d.copy_(lg_h, non_blocking=True)
            with torch.cuda.stream(pipe.down):
                y_h.copy_(y_d, non_blocking=True)
            torch.cuda.current_stream().wait_stream(pipe.up)
            torch.cuda.current_stream().wait_stream(pipe.down)

        c_ms = float(np.median(timed(copies_only, 5)))

        def copies_pattern():
            # the pipeline's own schedule with the layer left out: K uploads back to back on the up stream,
            # each batch's download on the down stream as soon as its upload is done
            a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a0.record(pipe.up)
            for i in range(args.steps):
                with torch.cuda.stream(pipe.up):
                    pipe.x[i % 2].copy_(x_h, non_blocking=True)
                    pipe.lg[i % 2].copy_(lg_h, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(pipe.up)
                pipe.down.wait_event(ev)
                with torch.cuda.stream(pipe.down):
                    ys_h[i % 2].copy_(pipe.y[i % 2], non_blocking=True)
            b0.record(pipe.down)
            torch.cuda.synchronize()
            return a0.elapsed_time(b0) / args.steps

        pat_ms = copies_pattern()
        line["e2e"]["roofline"] = {"bound": "pcie", "copies_only_ms": c_ms, "frac": c_ms / p_ms,
                                   "pattern_ms": pat_ms, "frac_of_pattern": pat_ms / p_ms,
                                   "note": "copies_only: one step's H2D and D2H bytes copied at once, nothing "
                                           "else; pattern: the pipeline's K-batch copy schedule without the "
                                           "layer (the bound the pipelined e2e number can reach on this box)"}
        del xd2

    if world > 1 and ep_mode == "peer" and not args.no_nccl_record:
        # the north star's NCCL all-to-all, measured beside the fused path on the same ranks and tokens: route +
        # one count exchange (host split sizes) + dispatch -> all_to_all_single -> grouped FFN ->
        # all_to_all_single -> combine, eager (split sizes are host values), max over ranks
        nl = ep.EPMoELayer.from_config(cfg, T, dist.group.WORLD, dev)
        for _ in range(args.warmup):
            nl.step()
        torch.cuda.synchronize()
        dist.barrier()
        n_ms = timed(nl.step, args.steps)
        dist.barrier()
        nt = torch.tensor([float(sum(n_ms))], device=dev)
        dist.all_reduce(nt, op=dist.ReduceOp.MAX)
        n_per = float(nt.item()) / args.steps
        line["nccl_exchange"] = {"value": T * world / (n_per * 1e-3), "unit": UNIT, "ms_per_step": n_per,
                                 "vs_fused": ms_per_step / n_per, "backend": dist.get_backend(),
                                 "mode": "NCCL all_to_all_single between the library's dispatch / grouped FFN / "
                                         "combine kernels, one count exchange per step, eager"}
        # what the fused path timed, checked: its last replay's output (y + residual, rounded once in the down
        # epilogue, in the arena) against the NCCL path on the same tokens (its combine adds the residual to the
        # bf16 y, a second rounding), per token: max |a - b|_inf / |b|_inf over rows and ranks against the
        # parity rule's 2e-2 (the two differ by the extra rounding: ~2^-8..2^-7 relative)
        y_nccl = nl.layer(residual=nl.x)
        torch.cuda.synchronize()
        a_, b_ = layer.out.float(), y_nccl.float()
        rel = ((a_ - b_).abs().amax(dim=1) / b_.abs().amax(dim=1).clamp_min(1e-6)).max()
        chk = torch.tensor([float(rel.item()), float((a_ - b_).abs().max().item()),
                            float(int(layer.dev_status.item()))], device=dev)
        dist.all_reduce(chk, op=dist.ReduceOp.MAX)
        line["ep_output_check"] = {"max_rel_err": float(chk[0].item()), "max_abs_diff": float(chk[1].item()),
                                   "tol": 2e-2, "ok": bool(chk[0].item() <= 2e-2 and chk[2].item() == 0),
                                   "dev_status": int(chk[2].item()),
                                   "what": "every rank's output rows of the timed fused peer-memory step vs the "
                                           "NCCL all-to-all path on the same tokens (per-token relative, max over "
                                           "rows and ranks)"}
        del nl
        torch.cuda.empty_cache()

    if world > 1 and not args.no_e2e:
        # e2e at N GPUs through the public API: every step each rank uploads its tokens and logits from
        # pinned host memory, runs the EP layer, and reads its output back; max over ranks
        lg_src = lg_ep if ep_mode == "peer" else layer.logits
        x_src = layer.x
        x_h = x_src.detach().cpu().pin_memory()
        lg_h = lg_src.detach().cpu().pin_memory()
        y_h = torch.empty_like(x_h).pin_memory()

        def e2e_step():
            x_src.copy_(x_h, non_blocking=True)
            lg_src.copy_(lg_h, non_blocking=True)
            out = eager_fn_out()
            y_h.copy_(out, non_blocking=True)

        def eager_fn_out():
            if ep_mode == "peer":
                layer.route(lg_src)
                return layer.layer(residual=True)
            return layer.step()

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        e_ms = timed(e2e_step, args.steps)
        dist.barrier()
        et = torch.tensor([float(sum(e_ms))], device=dev)
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_per = float(et.item()) / args.steps
        line["e2e"] = {"value": T * world / (e_per * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": (x_h.numel() * 2 + lg_h.numel() * lg_h.element_size()) * world,
                       "d2h_bytes_per_step": y_h.numel() * 2 * world, "ms_per_step": e_per,
                       "mode": "eager, one batch at a time per rank (H2D, route + EP layer, D2H)"}

    if world == 1:
        # the timed steps must not have flagged anything on the device (scheduler timeout, bad index, ...)
        st_timed = int(plan.dev_status.item())
        line["dev_status"] = st_timed
        if st_timed != 0:
            raise SystemExit(f"timed steps set dev_status = {st_timed:#x}: not reporting a number")
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"], sample, yref = cpu_baseline(cfg, inp)
        line["timed_output_check"] = timed_output_check(y, sample, yref, plan.dev_status)
        if not line["timed_output_check"]["ok"]:
            raise SystemExit(f"timed output check failed: {line['timed_output_check']}")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        if ep_mode == "peer":
            layer.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
