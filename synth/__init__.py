"""synth — seeded synthetic input generators shared by the tests, the bench and the oracle runs.

This module holds NONE of the method's arithmetic (no top-K, no grouping, no FFN): it only draws
random inputs with the shapes and distributions of the paper's workloads (recipe in DESIGN.md §Inputs).
Both the CUDA path (through tests/bench) and the oracle consume exactly the arrays it returns.

Generator: numpy's counter-based Philox bit generator, keyed per (master seed, tensor id, layer), so
every tensor is reproducible independently of the order in which tensors are drawn.
"""
from __future__ import annotations

import numpy as np

MASTER_SEED = 0x241019123

# tensor ids (layer l adds 16*l)
TID_X, TID_LOGITS, TID_WG, TID_WU, TID_WD, TID_NEURONS, TID_ASSIGN, TID_RESID = 1, 2, 3, 4, 5, 6, 7, 8

# BASELINE.json configs (the concrete synthetic recipe is SURVEY.md §8(d), restated in DESIGN.md).
CONFIGS = {
    1: dict(name="tiny", T=256, H=64, D=256, d=128, E=8, k=1, dtype="f32"),
    2: dict(name="prefill_layer", T=8192, H=4096, D=11008, d=5504, E=8, k=1, dtype="bf16"),
    3: dict(name="decode_batching", T=256, H=4096, D=11008, d=5504, E=8, k=1, dtype="bf16"),
    4: dict(name="stack32", T=16384, H=4096, D=11008, d=5504, E=8, k=1, dtype="bf16", L=32),
    5: dict(name="expert_parallel", T=65536, H=4096, D=11008, d=5504, E=8, k=1, dtype="bf16"),
}


def rng(seed: int, tensor_id: int, layer: int = 0) -> np.random.Generator:
    ss = np.random.SeedSequence([int(seed) & 0xFFFFFFFFFFFF, int(tensor_id) + 16 * int(layer)])
    return np.random.Generator(np.random.Philox(ss))


def normal(shape, seed: int, tensor_id: int, layer: int = 0, std: float = 1.0) -> np.ndarray:
    a = rng(seed, tensor_id, layer).standard_normal(size=shape, dtype=np.float32)
    if std != 1.0:
        a *= np.float32(std)
    return a


def tokens(T: int, H: int, seed: int = MASTER_SEED, layer: int = 0) -> np.ndarray:
    """x ~ N(0,1) [T,H] float32 (looks like post-RMSNorm hidden states)."""
    return normal((T, H), seed, TID_X, layer)


def residual(T: int, H: int, seed: int = MASTER_SEED, layer: int = 0) -> np.ndarray:
    return normal((T, H), seed, TID_RESID, layer)


def router_logits(T: int, E: int, seed: int = MASTER_SEED) -> np.ndarray:
    """i.i.d. N(0,1) gating logits [T,E] float32 -> near-uniform routing."""
    return normal((T, E), seed, TID_LOGITS)


def dense_ffn_weights(D: int, H: int, d: int, seed: int = MASTER_SEED, layer: int = 0):
    """Dense SwiGLU FFN: W_gate, W_up ~ N(0, 1/H) [D,H]; W_down ~ N(0, 1/d) [H,D] (float32)."""
    wg = normal((D, H), seed, TID_WG, layer, std=1.0 / np.sqrt(H))
    wu = normal((D, H), seed, TID_WU, layer, std=1.0 / np.sqrt(H))
    wd = normal((H, D), seed, TID_WD, layer, std=1.0 / np.sqrt(d))
    return wg, wu, wd


def expert_weights(E: int, d: int, H: int, seed: int = MASTER_SEED, layer: int = 0):
    """Expert stacks drawn directly (same distributions as slicing the dense weights):
    W_gate, W_up [E,d,H] ~ N(0,1/H); W_down [E,H,d] ~ N(0,1/d)."""
    wg = normal((E, d, H), seed, TID_WG + 100, layer, std=1.0 / np.sqrt(H))
    wu = normal((E, d, H), seed, TID_WU + 100, layer, std=1.0 / np.sqrt(H))
    wd = normal((E, H, d), seed, TID_WD + 100, layer, std=1.0 / np.sqrt(d))
    return wg, wu, wd


def expert_weights_device(E: int, d: int, H: int, device, seed: int = MASTER_SEED, layer: int = 0):
    """Same distributions as expert_weights(), drawn on the GPU with torch's Philox generator (used where a
    CPU draw would take minutes: the 32-layer stack has 17.3 G weights). bf16 [E,d,H], [E,d,H], [E,H,d]."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1000003 + 7919 * (layer + 1)) & 0x7FFFFFFFFFFFFFFF)
    out = []
    for shape, std in (((E, d, H), 1.0 / np.sqrt(H)), ((E, d, H), 1.0 / np.sqrt(H)), ((E, H, d), 1.0 / np.sqrt(d))):
        w = torch.randn(shape, generator=g, device=device, dtype=torch.float32).mul_(float(std))
        out.append(w.to(torch.bfloat16))
        del w
    return tuple(out)


def neuron_sets(E: int, D: int, d: int, seed: int = MASTER_SEED, mode: str = "overlap",
                layer: int = 0) -> np.ndarray:
    """Per-expert neuron lists S_e [E,d] int32, each strictly increasing.

    overlap: each expert keeps a random d-subset of [0,D) (d = D/2 by default);
    partition: a seeded permutation of [0,D) cut into E chunks of d = D/E (disjoint cover);
    full: every expert keeps all D neurons (d must equal D)."""
    g = rng(seed, TID_NEURONS, layer)
    if mode == "full":
        assert d == D
        return np.tile(np.arange(D, dtype=np.int32), (E, 1))
    if mode == "partition":
        assert E * d == D, "partition mode needs E*d == D"
        perm = g.permutation(D)
        return np.sort(perm.reshape(E, d), axis=1).astype(np.int32)
    out = np.empty((E, d), np.int32)
    for e in range(E):
        out[e] = np.sort(g.permutation(D)[:d])
    return out


def router_weights(vocab: int = 32000, n_experts: int = 8, seed: int = MASTER_SEED, dim: int = 512,
                   ffn: int = 512) -> dict:
    """Random-init pre-gating router (table:router_details): embeddings N(0,1), projections
    N(0, 1/fan_in) in nn.Linear [out, in] layout, RMSNorm weights 1 + 0.1 N(0,1), gating head N(0, 1/dim).
    float32 numpy arrays (callers round to bf16)."""
    tid = 200
    w = {
        "emb": normal((vocab, dim), seed, tid + 1),
        "norm1": 1.0 + normal((dim,), seed, tid + 2, std=0.1),
        "w_qkv": normal((3 * dim, dim), seed, tid + 3, std=1.0 / np.sqrt(dim)),
        "w_o": normal((dim, dim), seed, tid + 4, std=1.0 / np.sqrt(dim)),
        "norm2": 1.0 + normal((dim,), seed, tid + 5, std=0.1),
        "w_gate": normal((ffn, dim), seed, tid + 6, std=1.0 / np.sqrt(dim)),
        "w_up": normal((ffn, dim), seed, tid + 7, std=1.0 / np.sqrt(dim)),
        "w_down": normal((dim, ffn), seed, tid + 8, std=1.0 / np.sqrt(ffn)),
        "norm_f": 1.0 + normal((dim,), seed, tid + 9, std=0.1),
        "w_head": normal((n_experts, dim), seed, tid + 10, std=1.0 / np.sqrt(dim)),
    }
    return {k: v.astype(np.float32) for k, v in w.items()}


def token_ids(T: int, vocab: int = 32000, seed: int = MASTER_SEED) -> np.ndarray:
    """Synthetic token ids, Zipf-like over the vocabulary (a natural-text-like frequency profile)."""
    g = rng(seed, TID_ASSIGN + 40)
    r = g.zipf(1.2, size=T)
    return ((r - 1) % vocab).astype(np.int32)


# ---- routing-assignment recipes (the draws; turned into logits below) -------------------------------

def assignments_markov(n_req: int, req_len: int, E: int, p_follow: float = 0.672,
                       seed: int = MASTER_SEED) -> np.ndarray:
    """Temporal locality: each token keeps the previous token's expert with probability p_follow, else
    draws uniformly (p = 2921/4096 follow the previous token's expert)."""
    g = rng(seed, TID_ASSIGN)
    out = np.empty(n_req * req_len, np.int32)
    for r in range(n_req):
        cur = int(g.integers(E))
        follow = g.random(req_len) < p_follow
        fresh = g.integers(E, size=req_len)
        for i in range(req_len):
            if i > 0 and not follow[i]:
                cur = int(fresh[i])
            out[r * req_len + i] = cur
    return out


def assignments_zipf(B: int, E: int, s: float = 1.0, seed: int = MASTER_SEED) -> np.ndarray:
    """Zipf(s)-skewed expert ids over ranks 1..E, ranks -> ids through a seeded permutation."""
    g = rng(seed, TID_ASSIGN)
    ranks = np.arange(1, E + 1, dtype=np.float64)
    p = ranks ** (-s)
    p /= p.sum()
    perm = g.permutation(E)
    return perm[g.choice(E, size=B, p=p)].astype(np.int32)


def assignments_unique(B: int, u: int, E: int, seed: int = MASTER_SEED) -> np.ndarray:
    """B tokens drawn uniformly from exactly u distinct experts (each used at least once)."""
    g = rng(seed, TID_ASSIGN)
    experts = np.sort(g.permutation(E)[:u])
    ids = experts[g.integers(u, size=B)]
    ids[:u] = experts  # every chosen expert touched
    g.shuffle(ids)
    return ids.astype(np.int32)


def logits_for_assignments(ids: np.ndarray, E: int, margin: float = 0.5,
                           seed: int = MASTER_SEED) -> np.ndarray:
    """Logits whose largest entry sits at ids[t], at least `margin` above the runner-up."""
    lg = normal((ids.shape[0], E), seed, TID_LOGITS)
    rows = np.arange(ids.shape[0])
    lg[rows, ids] = -np.inf
    top = lg.max(axis=1)
    top[~np.isfinite(top)] = 0.0  # E == 1: no runner-up
    lg[rows, ids] = top + np.float32(margin) + np.abs(normal((ids.shape[0],), seed, TID_LOGITS + 50))
    return lg.astype(np.float32)


def near_tie_logits(T: int, E: int, seed: int = MASTER_SEED) -> np.ndarray:
    """N(0,1) logits with injected exact ties, 1-ulp margins, signed zeros and long equal rows."""
    lg = normal((T, E), seed, TID_LOGITS + 7)
    g = rng(seed, TID_LOGITS + 8)
    n = max(1, T // 8)
    rows = g.choice(T, size=min(T, 4 * n), replace=False)
    for i, t in enumerate(rows):
        a, b = g.choice(E, size=2, replace=False) if E > 1 else (0, 0)
        kind = i % 4
        if kind == 0:  # exact tie at the top
            lg[t, b] = lg[t, a] = lg[t].max() + 1.0
        elif kind == 1:  # 1-ulp margin at the top
            top = np.float32(lg[t].max() + 1.0)
            lg[t, a] = top
            lg[t, b] = np.nextafter(top, np.float32(-np.inf))
        elif kind == 2:  # all equal
            lg[t, :] = np.float32(0.25)
        else:  # signed zeros as the maximum
            lg[t, :] = -np.abs(lg[t, :]) - 1.0
            lg[t, a] = np.float32(-0.0)
            lg[t, b] = np.float32(0.0)
    return lg.astype(np.float32)


# ---- dtype helpers ----------------------------------------------------------------------------------

def to_torch(a: np.ndarray, dtype: str = "bf16"):
    """float32 numpy -> torch CPU tensor of the storage dtype ('bf16' rounds RNE, 'f32' exact)."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype == "bf16":
        return t.to(torch.bfloat16)
    if dtype == "f32":
        return t.to(torch.float32)
    raise ValueError(dtype)
