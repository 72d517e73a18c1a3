"""Expert parallelism over one NVLink/NVSwitch box: experts sharded by GPU, tokens
data-parallel, dispatch/combine as NCCL all-to-all.

Partitioning: rank r holds its own batch of T_r tokens and routes them locally with the (replicated)
pre-gating logits; rank q owns experts [q*E/G, (q+1)*E/G) and only their weights. Because the router is
independent of the layer, the per-destination split sizes are fixed for the
whole batch: ONE count exchange (C1) per batch, then per layer one all-to-all each way (C2 dispatch,
C3 combine). This is the system advantage the paper claims over layer-wise routers.

Local route sorts rows by expert, which (experts contiguous per rank) is already by destination rank, so
the send buffer is x_sorted itself. Rows arrive in source-rank order; the receive buffer is therefore
G groups of E_local segments, segment g -> local expert g % E_local, which readme_expert_ffn takes
directly through its n_src argument (no second local permutation). Each expert's rows arrive in global
token order, so EP output equals the single-GPU output bit for bit (P12).

Host logic (plan_from_counts, exchange) is device-agnostic and is exercised with gloo on CPU in
tests/test_ep_gloo.py; the GPU layer (EPMoELayer) runs every compute step in libreadme_b200 kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class EPPlan:
    G: int
    rank: int
    E: int
    E_local: int
    send_splits: list      # rows this rank sends to each rank q (= its rows for q's experts)
    recv_splits: list      # rows this rank receives from each source p
    recv_counts: np.ndarray  # [G, E_local] rows from source p for local expert e
    seg_offsets: np.ndarray  # [G*E_local + 1] exclusive scan of recv_counts (source-major)

    @property
    def rows_in(self) -> int:
        return int(self.seg_offsets[-1])


def _host_staged(group) -> bool:
    """gloo has no device all-to-all: stage CUDA tensors through host memory (CPU tests, one-GPU tests)."""
    return dist.get_backend(group) == "gloo"


def plan_from_counts(counts_local, group=None) -> EPPlan:
    """C1: exchange per-expert counts once per batch. `counts_local` is this rank's [E] int32 histogram
    (any device the process group's backend accepts). Returns host-side split lists and segment table."""
    G = dist.get_world_size(group)
    rank = dist.get_rank(group)
    E = counts_local.numel()
    if E % G:
        raise ValueError(f"E={E} experts cannot be sharded over {G} ranks")
    El = E // G
    send = counts_local.reshape(G, El).contiguous()
    if _host_staged(group):
        send = send.cpu()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)  # recv[p, e] = rows source p has for my expert e
    send_h = send.cpu().numpy().astype(np.int64)
    recv_h = recv.cpu().numpy().astype(np.int64)
    seg = np.zeros(G * El + 1, np.int64)
    seg[1:] = np.cumsum(recv_h.reshape(-1))
    return EPPlan(G=G, rank=rank, E=E, E_local=El, send_splits=send_h.sum(axis=1).tolist(),
                  recv_splits=recv_h.sum(axis=1).tolist(), recv_counts=recv_h, seg_offsets=seg)


def exchange(rows: torch.Tensor, plan: EPPlan, reverse: bool = False, out: torch.Tensor | None = None,
             group=None) -> torch.Tensor:
    """C2 (dispatch, reverse=False): send my expert-sorted rows to their experts' owners, receive rows in
    source-rank order. C3 (combine, reverse=True): the mirror image."""
    in_s, out_s = (plan.recv_splits, plan.send_splits) if reverse else (plan.send_splits, plan.recv_splits)
    n_out = int(sum(out_s))
    if out is None:
        out = torch.empty((n_out,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    if _host_staged(group) and rows.is_cuda:
        tmp = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(tmp, rows.cpu(), output_split_sizes=out_s, input_split_sizes=in_s, group=group)
        out.copy_(tmp)
        return out
    dist.all_to_all_single(out, rows, output_split_sizes=out_s, input_split_sizes=in_s, group=group)
    return out


class EPMoELayer:
    """One expert-parallel pre-gated MoE layer on this rank's GPU (NCCL process group)."""

    def __init__(self, x, logits, w_gate, w_up, w_down, E: int, k: int, group=None):
        from . import readme as rd
        self.rd = rd
        self.group = group
        self.x, self.logits = x, logits
        self.w = (w_gate, w_up, w_down)
        self.E, self.k = E, k
        T, H = x.shape
        self.T, self.H = T, H
        self.d = w_gate.shape[1]
        dev = x.device
        self.plan = rd.new_plan(T, E, k, dev)
        self.ws_r = torch.empty(rd.route_workspace_bytes(T, E, k), dtype=torch.uint8, device=dev)
        self.xs = torch.empty((T * k, H), dtype=x.dtype, device=dev)
        self.ys = torch.empty_like(self.xs)
        self.y = torch.empty_like(x)
        self.ep = None

    @classmethod
    def from_config(cls, cfg: dict, T: int, group, device):
        """Synthetic config-5 layer: this rank's tokens/logits and its shard of the experts."""
        import synth
        from . import readme as rd
        G, rank = dist.get_world_size(group), dist.get_rank(group)
        H, D, d, E, k = cfg["H"], cfg["D"], cfg["d"], cfg["E"], cfg["k"]
        El = E // G
        seed = synth.MASTER_SEED + 5
        wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=seed)
        S = synth.neuron_sets(E, D, d, seed=seed)[rank * El:(rank + 1) * El]
        dense = [synth.to_torch(w, "bf16").to(device) for w in (wg, wu, wd)]
        del wg, wu, wd
        eg, eu, ed = rd.build_experts(*dense, torch.from_numpy(np.ascontiguousarray(S)).to(device))
        del dense
        x = synth.to_torch(synth.tokens(T, H, seed=seed + 1000 * rank), "bf16").to(device)
        lg = torch.from_numpy(synth.router_logits(T, E, seed=seed + 1000 * rank)).to(device)
        return cls(x, lg, eg, eu, ed, E, k, group)

    def route(self):
        """Once per batch: local routing plan + C1 count exchange (the only device->host sync)."""
        self.rd.route(self.logits, self.k, plan=self.plan, ws=self.ws_r)
        self.ep = plan_from_counts(self.plan.counts, self.group)
        self.seg_dev = torch.from_numpy(self.ep.seg_offsets.astype(np.int32)).to(self.x.device)
        rows = self.ep.rows_in
        self.x_recv = torch.empty((rows, self.H), dtype=self.x.dtype, device=self.x.device)
        self.y_recv = torch.empty_like(self.x_recv)
        self.ws_f = torch.empty(self.rd.expert_ffn_workspace_bytes(max(rows, 1), self.H, self.ep.E_local, self.d,
                                                                   self.x.dtype), dtype=torch.uint8,
                                device=self.x.device)

    def layer(self, x=None, residual=None):
        """Per layer (plan reused): dispatch -> C2 -> grouped FFN over (source, local expert) segments -> C3
        -> combine."""
        rd, ep = self.rd, self.ep
        x = self.x if x is None else x
        rd.dispatch(x, self.plan.dest, self.k, out=self.xs)
        exchange(self.xs, ep, out=self.x_recv, group=self.group)
        if ep.rows_in:
            rd.expert_ffn(self.x_recv, self.seg_dev, *self.w, n_src=ep.G, out=self.y_recv, ws=self.ws_f)
        exchange(self.y_recv, ep, reverse=True, out=self.ys, group=self.group)
        return rd.combine(self.ys, self.plan.dest, self.plan.topk_w, self.k, residual=residual, out=self.y)

    def step(self):
        self.route()
        return self.layer()


# ---- the fused path: expert parallelism over peer memory (readme_ep_*) ---------------------------------

class PeerArena:
    """Symmetric device memory: one library-owned block per rank (readme_ep_alloc), mapped into every other
    rank of `group` with CUDA IPC (readme_ipc_handle/readme_ipc_open; on NVLink/NVSwitch the mapping is a
    peer mapping, on one GPU shared by several processes it is the same device memory). `layout` maps
    names to (shape, dtype); every rank uses the same layout, so region r of rank q sits at
    base[q] + offset[r]."""

    def __init__(self, layout: dict, group, device):
        from . import readme as rd
        self.rd = rd
        self.group = group
        self.G, self.me = dist.get_world_size(group), dist.get_rank(group)
        self.device = torch.device(device)
        self.off, self.spec, off = {}, {}, 0
        for name, (shape, dtype) in layout.items():
            nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
            self.off[name], self.spec[name] = off, (tuple(shape), dtype)
            off += (nbytes + 255) // 256 * 256
        self.nbytes = max(off, 256)
        self.base_own = rd.ep_alloc(self.nbytes, self.device)
        handles = [None] * self.G
        dist.all_gather_object(handles, rd.ipc_handle(self.base_own), group=group)
        self.base = [self.base_own if q == self.me else rd.ipc_open(handles[q], self.device) for q in range(self.G)]
        self.t = {name: rd.device_view(self.base_own + self.off[name], *self.spec[name], self.device)
                  for name in layout}

    def peers(self, name: str, extra_bytes: int = 0):
        return [b + self.off[name] + extra_bytes for b in self.base]

    def close(self):
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for q, b in enumerate(self.base):
            if q != self.me:
                self.rd.ipc_close(b)
        dist.barrier(group=self.group)
        self.rd.ep_free(self.base_own)
        self.base = []


class PeerEPLayer:
    """One expert-parallel pre-gated MoE layer with the all-to-alls fused into the kernels (SURVEY §8(e),
    stretch C4): readme_ep_dispatch stores each token row into its expert owner's receive buffer,
    readme_ep_expert_ffn's down epilogue stores each result row (+ the source's residual, k == 1) into the
    source rank's output, and system-scope flag words order the phases. Once per batch (route): counts to
    every peer and the receive layout (readme_ep_publish_counts / readme_ep_plan), no host round trip.

    Inputs live in the arena: write this rank's tokens into `self.x` (or run layers back to back: the
    output is returned as a view of the arena and can be copied into `self.x`)."""

    A, B, C = 0, 1, 2  # phases: counts published, rows delivered, results returned

    def __init__(self, T: int, H: int, E: int, k: int, w_gate, w_up, w_down, group=None, device=None):
        from . import readme as rd
        self.rd = rd
        self.group = group
        self.G, self.me = dist.get_world_size(group), dist.get_rank(group)
        if E % self.G:
            raise ValueError(f"E={E} experts cannot be sharded over {self.G} ranks")
        self.T, self.H, self.E, self.k = T, H, E, k
        self.El = E // self.G
        self.w = (w_gate, w_up, w_down)
        self.d = w_gate.shape[1]
        dev = torch.device(device) if device is not None else w_gate.device
        self.dev = dev
        G, El = self.G, self.El
        self.rows_cap = G * T * k               # worst case: every token of every rank picks my experts
        self.vrows = T if k == 1 else T * k     # k == 1: rows return to y[t]; else to y_sorted[r]
        bf = torch.bfloat16
        self.arena = PeerArena({
            "flags": ((3, G), torch.int64), "table": ((G, E), torch.int32),
            "seg": ((G * El + 1,), torch.int32), "row_base": ((E,), torch.int32),
            "row_map": ((self.rows_cap,), torch.int32), "x": ((T, H), bf), "out": ((self.vrows, H), bf),
            "x_recv": ((self.rows_cap, H), bf)}, group, dev)
        t = self.arena.t
        self.x, self.out = t["x"], t["out"]
        self.plan = rd.new_plan(T, E, k, dev)
        self.ws_r = torch.empty(rd.route_workspace_bytes(T, E, k), dtype=torch.uint8, device=dev)
        self.ws_f = torch.empty(rd.expert_ffn_workspace_bytes(self.rows_cap, H, El, self.d, bf), dtype=torch.uint8,
                                device=dev)
        self.y = torch.empty((T, H), dtype=bf, device=dev) if k > 1 else None
        self.dev_status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epochs = torch.zeros(3, dtype=torch.int64, device=dev)  # this rank's phase counters

    @classmethod
    def from_config(cls, cfg: dict, T: int, group, device):
        """Synthetic config-5 layer (as EPMoELayer.from_config): returns (layer, logits); x is in the arena."""
        import synth
        from . import readme as rd
        G, rank = dist.get_world_size(group), dist.get_rank(group)
        H, D, d, E, k = cfg["H"], cfg["D"], cfg["d"], cfg["E"], cfg["k"]
        El = E // G
        seed = synth.MASTER_SEED + 5
        wg, wu, wd = synth.dense_ffn_weights(D, H, d, seed=seed)
        S = synth.neuron_sets(E, D, d, seed=seed)[rank * El:(rank + 1) * El]
        dense = [synth.to_torch(w, "bf16").to(device) for w in (wg, wu, wd)]
        del wg, wu, wd
        eg, eu, ed = rd.build_experts(*dense, torch.from_numpy(np.ascontiguousarray(S)).to(device))
        del dense
        layer = cls(T, H, E, k, eg, eu, ed, group, device)
        layer.x.copy_(synth.to_torch(synth.tokens(T, H, seed=seed + 1000 * rank), "bf16").to(device))
        lg = torch.from_numpy(synth.router_logits(T, E, seed=seed + 1000 * rank)).to(device)
        return layer, lg

    def _flags(self, phase: int):
        return self.arena.peers("flags", phase * self.G * 8)

    def _sync(self, phase: int):
        """Signal my arrival at `phase` to every rank, then wait until every rank has arrived (device-side
        epochs: no host value is baked in, so a captured graph of a layer replays correctly)."""
        epoch = self.epochs.data_ptr() + phase * 8
        self.rd.ep_signal(self._flags(phase), self.me, epoch, self.dev)
        self.rd.ep_wait(self.arena.base_own + self.arena.off["flags"] + phase * self.G * 8, self.G, epoch,
                        self.dev_status, self.dev)

    def route(self, logits):
        """Once per batch: local plan, counts to every peer, receive layout and row bases (device only)."""
        rd, a = self.rd, self.arena
        rd.route(logits, self.k, plan=self.plan, ws=self.ws_r)
        rd.ep_publish_counts(self.plan.counts, a.peers("table"), self.me)
        self._sync(self.A)
        rd.ep_plan(a.base_own + a.off["table"], self.G, self.E, self.me, a.t["seg"], a.t["row_base"])

    def layer(self, residual: bool = True):
        """dispatch (+ all-to-all) -> grouped FFN (+ reverse all-to-all, + residual for k == 1) [-> combine]."""
        rd, a, p = self.rd, self.arena, self.plan
        k1 = self.k == 1
        rd.ep_dispatch(self.x, self.k, p.dest, p.offsets, a.t["row_base"], self.E, self.me, a.peers("x_recv"),
                       a.peers("row_map"), self.vrows, k1, self.dev_status)
        self._sync(self.B)
        rd.ep_expert_ffn(a.t["x_recv"], a.t["seg"], *self.w, a.t["row_map"], a.peers("out"),
                         a.peers("x") if (k1 and residual) else None, self.vrows, self.ws_f, self.dev_status)
        self._sync(self.C)
        if k1:
            return self.out
        return rd.combine(self.out, p.dest, p.topk_w, self.k, residual=self.x if residual else None, out=self.y)

    def close(self):
        self.arena.close()
