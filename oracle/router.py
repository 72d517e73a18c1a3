"""oracle.router — TEST INFRASTRUCTURE ONLY. The pre-gating router G (§2.3; table:router_details,
PAPER.md:276-294), written in plain numpy float64, for checking readme_router_forward.

G(x_<=t): one causal transformer block (4 heads x 128, dim 512, SwiGLU MLP 512, RoPE, RMSNorm) over the
token embeddings, then a linear gating head to N expert logits. Readings (Q15): pre-norm block
    h0 = Emb[ids];  h1 = h0 + Attn(RMSNorm(h0; g1));  h2 = h1 + W_d(silu(W_g m) * (W_u m)), m = RMSNorm(h1; g2)
    logits = RMSNorm(h2; gf) W_head^T
RMSNorm(x; g) = x / sqrt(mean(x^2) + eps) * g; RoPE rotates dims (i, i+64) of each head by pos * 10000^(-2i/128);
attention is causal within each sequence and positions restart at 0 per sequence. Inputs bf16 are widened
exactly to float64; nothing is rounded.

Two independent evaluations are provided: `forward` (masked full-sequence matrices) and
`forward_incremental` (token by token with a growing key/value cache — no mask at all); tests check they
agree, which pins the causal mask and the RoPE positions.
"""
from __future__ import annotations

import numpy as np

D, HEADS, HD, THETA = 512, 4, 128, 10000.0
KEYS = ("emb", "norm1", "w_qkv", "w_o", "norm2", "w_gate", "w_up", "w_down", "norm_f", "w_head")


def _f64(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().double().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(a, dtype=np.float64)


def rmsnorm(x, g, eps):
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope(x, pos):
    """x [n, 128] (one head), pos [n] -> rotated copy."""
    i = np.arange(HD // 2, dtype=np.float64)
    ang = pos[:, None].astype(np.float64) * THETA ** (-2.0 * i / HD)[None, :]
    c, s = np.cos(ang), np.sin(ang)
    lo, hi = x[:, :HD // 2], x[:, HD // 2:]
    return np.concatenate([lo * c - hi * s, hi * c + lo * s], axis=1)


def silu(z):
    return z / (1.0 + np.exp(-z))


def param_count(W) -> int:
    return int(sum(np.asarray(_f64(W[k])).size for k in KEYS))


def _mlp_and_head(h1, W, eps):
    m = rmsnorm(h1, W["norm2"], eps)
    h2 = h1 + (silu(m @ W["w_gate"].T) * (m @ W["w_up"].T)) @ W["w_down"].T
    return rmsnorm(h2, W["norm_f"], eps) @ W["w_head"].T


def forward(ids, seq_starts, weights, eps: float = 1e-5):
    """Masked whole-sequence evaluation. Returns logits [T, N] float64."""
    W = {k: _f64(weights[k]) for k in KEYS}
    ids = np.asarray(ids, dtype=np.int64)
    h0 = W["emb"][ids]
    a = rmsnorm(h0, W["norm1"], eps)
    qkv = a @ W["w_qkv"].T
    att = np.zeros_like(h0)
    st = list(np.asarray(seq_starts))
    for s0, s1 in zip(st[:-1], st[1:]):
        n = s1 - s0
        if n == 0:
            continue
        pos = np.arange(n)
        mask = np.tril(np.ones((n, n), dtype=bool))
        for h in range(HEADS):
            q = rope(qkv[s0:s1, h * HD:(h + 1) * HD], pos)
            k = rope(qkv[s0:s1, D + h * HD:D + (h + 1) * HD], pos)
            v = qkv[s0:s1, 2 * D + h * HD:2 * D + (h + 1) * HD]
            sc = np.where(mask, (q @ k.T) / np.sqrt(HD), -np.inf)
            p = np.exp(sc - sc.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            att[s0:s1, h * HD:(h + 1) * HD] = p @ v
    h1 = h0 + att @ W["w_o"].T
    return _mlp_and_head(h1, W, eps)


def forward_incremental(ids, seq_starts, weights, eps: float = 1e-5):
    """Token-by-token evaluation with a growing key/value cache (no mask): logits [T, N] float64."""
    W = {k: _f64(weights[k]) for k in KEYS}
    ids = np.asarray(ids, dtype=np.int64)
    out = np.zeros((ids.size, W["w_head"].shape[0]))
    st = list(np.asarray(seq_starts))
    for s0, s1 in zip(st[:-1], st[1:]):
        ks = [[] for _ in range(HEADS)]
        vs = [[] for _ in range(HEADS)]
        for t in range(s0, s1):
            p = t - s0
            h0 = W["emb"][ids[t]][None, :]
            qkv = rmsnorm(h0, W["norm1"], eps) @ W["w_qkv"].T
            o = np.zeros((1, D))
            for h in range(HEADS):
                q = rope(qkv[:, h * HD:(h + 1) * HD], np.array([p]))[0]
                ks[h].append(rope(qkv[:, D + h * HD:D + (h + 1) * HD], np.array([p]))[0])
                vs[h].append(qkv[0, 2 * D + h * HD:2 * D + (h + 1) * HD])
                sc = np.array([q @ kk for kk in ks[h]]) / np.sqrt(HD)
                w = np.exp(sc - sc.max())
                w /= w.sum()
                o[0, h * HD:(h + 1) * HD] = sum(wi * vi for wi, vi in zip(w, vs[h]))
            h1 = h0 + o @ W["w_o"].T
            out[t] = _mlp_and_head(h1, W, eps)[0]
    return out
