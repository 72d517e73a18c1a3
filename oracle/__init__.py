"""oracle — TEST INFRASTRUCTURE ONLY (not the product path).

A plain, slow fp64 CPU implementation of READ-ME's pre-gated MoE layer (arXiv 2410.19123, Eq. 2,
PAPER.md:136-138; expert definition; route once for all layers PAPER.md:140-142, :237),
written in C++17 (oracle/oracle.cpp) and wrapped here with ctypes + numpy.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. It shares no code with ``paper_2410_19123_b200`` and
the CUDA path never calls it.

Inputs may be float64, float32 or bfloat16 (passed as uint16 bit patterns); the C code widens each
element exactly to double. Outputs are float64 (values) and int32 (routing plan).

Pins: see the header of oracle.cpp and tests/test_oracle_pins.py. Parity unpinned: the realism of the
synthetic inputs (no checkpoint or trained router exists here).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

DT_F64, DT_F32, DT_BF16 = 0, 1, 2
OK, BAD_ARG, NONFINITE = 0, 1, 2


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (g++ -O2, no fast-math, no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
                               "-fno-fast-math", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            _lib = ctypes.CDLL(_LIB)
    return _lib


def _as_input(a):
    """numpy/torch array -> (contiguous numpy array, dtype code)."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            a = a.detach().cpu().contiguous()
            if a.dtype == torch.bfloat16:
                return a.view(torch.int16).numpy().view(np.uint16), DT_BF16
            a = a.numpy()
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        return a, DT_F64
    if a.dtype == np.float32:
        return a, DT_F32
    if a.dtype == np.uint16:  # raw bf16 bits
        return a, DT_BF16
    raise TypeError(f"oracle input dtype {a.dtype} not supported")


def _weights(*ws):
    """Convert a group of weight arrays to one common dtype code (upcast to f64 if they differ)."""
    conv = [_as_input(w) for w in ws]
    if len({dt for _, dt in conv}) == 1:
        return [a for a, _ in conv], conv[0][1]
    out = []
    for w in ws:
        try:
            import torch
            if isinstance(w, torch.Tensor):
                w = w.detach().cpu().double().numpy()
        except ImportError:  # pragma: no cover
            pass
        out.append(np.ascontiguousarray(w, dtype=np.float64))
    return out, DT_F64


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc == NONFINITE:
        raise OracleError(f"{what}: non-finite logit (SPEC.md:167)")
    if rc != OK:
        raise OracleError(f"{what}: bad argument (rc={rc})")


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def route(logits, k: int):
    """a1-a4: top-K ids (descending logit, ties -> lower id), softmax-over-selected weights, counts,
    offsets (exclusive scan), dest (stable slot -> row) and src = dest^-1."""
    lib = _load()
    lg, ldt = _as_input(logits)
    T, E = lg.shape
    idx = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float64)
    counts = np.empty(E, np.int32)
    offsets = np.empty(E + 1, np.int32)
    dest = np.empty(T * k, np.int32)
    src = np.empty(T * k, np.int32)
    rc = lib.oracle_route(_p(lg), ctypes.c_int32(ldt), ctypes.c_int64(T), ctypes.c_int32(E),
                          ctypes.c_int32(k), _p(idx), _p(w), _p(counts), _p(offsets), _p(dest), _p(src))
    _check(rc, "oracle_route")
    return dict(topk_idx=idx, topk_w=w, counts=counts, offsets=offsets, dest=dest, src=src)


def dispatch(x, dest, k: int):
    """a5: x_sorted[dest[s]] = x[s // k] (fp64 copy)."""
    lib = _load()
    xa, xdt = _as_input(x)
    T, H = xa.shape
    dest = _i32(dest)
    out = np.empty((T * k, H), np.float64)
    rc = lib.oracle_dispatch(_p(xa), ctypes.c_int32(xdt), ctypes.c_int64(T), ctypes.c_int32(H),
                             ctypes.c_int32(k), _p(dest), _p(out))
    _check(rc, "oracle_dispatch")
    return out


def expert_ffn(x_sorted, offsets, w_gate, w_up, w_down, n_src: int = 1, act: str = "swiglu",
               nthreads: int | None = None):
    """a6+a7: per-segment expert FFN; segment g uses expert g % E. Returns y_sorted fp64 [rows, H]."""
    lib = _load()
    xa, xdt = _as_input(x_sorted)
    rows, H = xa.shape
    (wg, wu, wd), wdt = _weights(w_gate, w_up, w_down)
    E, d, H2 = wg.shape
    assert H2 == H and wd.shape == (E, H, d)
    offsets = _i32(offsets)
    assert offsets.shape == (n_src * E + 1,)
    out = np.empty((rows, H), np.float64)
    rc = lib.oracle_expert_ffn(_p(xa), ctypes.c_int32(xdt), ctypes.c_int64(rows), ctypes.c_int32(H),
                               ctypes.c_int32(E), ctypes.c_int32(d), ctypes.c_int32(n_src), _p(offsets),
                               _p(wg), _p(wu), _p(wd), ctypes.c_int32(wdt),
                               ctypes.c_int32(0 if act == "swiglu" else 1), _p(out),
                               ctypes.c_int32(nthreads or default_threads()))
    _check(rc, "oracle_expert_ffn")
    return out


def expert_hidden(x_sorted, offsets, w_gate, w_up, n_src: int = 1, nthreads: int | None = None):
    """a6 alone: h = silu(x W_gate[e]^T) * (x W_up[e]^T), fp64 [rows, d]."""
    lib = _load()
    xa, xdt = _as_input(x_sorted)
    rows, H = xa.shape
    (wg, wu), wdt = _weights(w_gate, w_up)
    E, d, _ = wg.shape
    offsets = _i32(offsets)
    out = np.empty((rows, d), np.float64)
    rc = lib.oracle_expert_hidden(_p(xa), ctypes.c_int32(xdt), ctypes.c_int64(rows), ctypes.c_int32(H),
                                  ctypes.c_int32(E), ctypes.c_int32(d), ctypes.c_int32(n_src), _p(offsets), _p(wg),
                                  _p(wu), ctypes.c_int32(wdt), _p(out), ctypes.c_int32(nthreads or default_threads()))
    _check(rc, "oracle_expert_hidden")
    return out


def expert_down(h, offsets, w_down, n_src: int = 1, nthreads: int | None = None):
    """a7 alone: y = h W_down[e]^T, fp64 [rows, H]."""
    lib = _load()
    ha, hdt = _as_input(h)
    rows, d = ha.shape
    wd, wdt = _as_input(w_down)
    E, H, _ = wd.shape
    offsets = _i32(offsets)
    out = np.empty((rows, H), np.float64)
    rc = lib.oracle_expert_down(_p(ha), ctypes.c_int32(hdt), ctypes.c_int64(rows), ctypes.c_int32(H),
                                ctypes.c_int32(E), ctypes.c_int32(d), ctypes.c_int32(n_src), _p(offsets), _p(wd),
                                ctypes.c_int32(wdt), _p(out), ctypes.c_int32(nthreads or default_threads()))
    _check(rc, "oracle_expert_down")
    return out


def rmsnorm(x, eps: float = 1e-5):
    """RMSNorm with weight 1 (reading Q10): x / sqrt(mean(x^2) + eps), fp64."""
    lib = _load()
    xa, xdt = _as_input(x)
    T, H = xa.shape
    out = np.empty((T, H), np.float64)
    rc = lib.oracle_rmsnorm(_p(xa), ctypes.c_int32(xdt), ctypes.c_int64(T), ctypes.c_int32(H), ctypes.c_double(eps),
                            _p(out))
    _check(rc, "oracle_rmsnorm")
    return out


def moe_stack(x, logits, k: int, layers, eps: float = 1e-5, nthreads: int | None = None):
    """Config 4: x <- x + MoE_l(RMSNorm(x)) for each layer, routed ONCE from the pre-gating logits
    (PAPER.md:140-142, :237). `layers` = [(w_gate, w_up, w_down), ...]. Returns (x fp64, plan)."""
    plan = route(logits, k)
    xa, _ = _as_input(x)
    xd = np.array(xa if xa.dtype != np.uint16 else _bf16_to_f64(xa), dtype=np.float64)
    for (wg, wu, wd) in layers:
        xs = dispatch(rmsnorm(xd, eps), plan["dest"], k)
        ys = expert_ffn(xs, plan["offsets"], wg, wu, wd, nthreads=nthreads)
        xd = combine(ys, plan["dest"], plan["topk_w"], k, residual=xd)
    return xd, plan


def _bf16_to_f64(a):
    return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def combine(y_sorted, dest, topk_w, k: int, residual=None):
    """a8: y[t] = res[t] + sum_j w[t,j] * y_sorted[dest[t*k+j]] (j ascending)."""
    lib = _load()
    ys = np.ascontiguousarray(y_sorted, dtype=np.float64)
    rows, H = ys.shape
    T = rows // k
    dest = _i32(dest)
    w = np.ascontiguousarray(topk_w, dtype=np.float64).reshape(T, k)
    ra, rdt = (None, 0) if residual is None else _as_input(residual)
    out = np.empty((T, H), np.float64)
    rc = lib.oracle_combine(_p(ys), ctypes.c_int64(T), ctypes.c_int32(H), ctypes.c_int32(k), _p(dest),
                            _p(w), _p(ra), ctypes.c_int32(rdt), _p(out))
    _check(rc, "oracle_combine")
    return out


def moe_layer(x, logits, k: int, w_gate, w_up, w_down, residual=None, act: str = "swiglu",
              nthreads: int | None = None):
    """Eq. 2 for one layer: route -> dispatch -> expert FFN -> combine. Returns (y, plan dict)."""
    lib = _load()
    xa, xdt = _as_input(x)
    lg, ldt = _as_input(logits)
    (wg, wu, wd), wdt = _weights(w_gate, w_up, w_down)
    T, H = xa.shape
    E, d, _H = wg.shape
    ra, rdt = (None, 0) if residual is None else _as_input(residual)
    y = np.empty((T, H), np.float64)
    idx = np.empty((T, k), np.int32)
    w = np.empty((T, k), np.float64)
    counts = np.empty(E, np.int32)
    offsets = np.empty(E + 1, np.int32)
    dest = np.empty(T * k, np.int32)
    src = np.empty(T * k, np.int32)
    rc = lib.oracle_moe_layer(_p(xa), ctypes.c_int32(xdt), ctypes.c_int64(T), ctypes.c_int32(H), _p(lg),
                              ctypes.c_int32(ldt), ctypes.c_int32(E), ctypes.c_int32(k), ctypes.c_int32(d),
                              _p(wg), _p(wu), _p(wd), ctypes.c_int32(wdt),
                              ctypes.c_int32(0 if act == "swiglu" else 1), _p(ra), ctypes.c_int32(rdt),
                              _p(y), _p(idx), _p(w), _p(counts), _p(offsets), _p(dest), _p(src),
                              ctypes.c_int32(nthreads or default_threads()))
    _check(rc, "oracle_moe_layer")
    return y, dict(topk_idx=idx, topk_w=w, counts=counts, offsets=offsets, dest=dest, src=src)


def dense_ffn(x, wg, wu, wd, act: str = "swiglu", nthreads: int | None = None):
    """F_0(x) = W_2 sigma(W_1 x) on the dense [D,H] / [H,D] weights."""
    lib = _load()
    xa, xdt = _as_input(x)
    (ga, ua, da), wdt = _weights(wg, wu, wd)
    T, H = xa.shape
    D = ga.shape[0]
    y = np.empty((T, H), np.float64)
    rc = lib.oracle_dense_ffn(_p(xa), ctypes.c_int32(xdt), ctypes.c_int64(T), ctypes.c_int32(H),
                              ctypes.c_int32(D), _p(ga), _p(ua), _p(da), ctypes.c_int32(wdt),
                              ctypes.c_int32(0 if act == "swiglu" else 1), _p(y),
                              ctypes.c_int32(nthreads or default_threads()))
    _check(rc, "oracle_dense_ffn")
    return y


def build_experts(wg, wu, wd, neuron_idx):
    """Expert slicing: rows S_e of W_gate/W_up, columns S_e of W_down."""
    lib = _load()
    (ga, ua, da), wdt = _weights(wg, wu, wd)
    D, H = ga.shape
    nidx = _i32(neuron_idx)
    E, d = nidx.shape
    eg = np.empty((E, d, H), np.float64)
    eu = np.empty((E, d, H), np.float64)
    ed = np.empty((E, H, d), np.float64)
    rc = lib.oracle_build_experts(_p(ga), _p(ua), _p(da), ctypes.c_int32(wdt), ctypes.c_int32(D),
                                  ctypes.c_int32(H), ctypes.c_int32(E), ctypes.c_int32(d), _p(nidx),
                                  _p(eg), _p(eu), _p(ed))
    _check(rc, "oracle_build_experts")
    return eg, eu, ed


def bruteforce(x, logits, k: int, wg, wu, wd, neuron_idx, act: str = "swiglu"):
    """Eq. 2 literally, per token, from the dense weights and neuron lists (no sort/scan/buffers)."""
    lib = _load()
    xa, xdt = _as_input(x)
    lg, ldt = _as_input(logits)
    (ga, ua, da), wdt = _weights(wg, wu, wd)
    T, H = xa.shape
    E = lg.shape[1]
    D = ga.shape[0]
    nidx = _i32(neuron_idx)
    d = nidx.shape[1]
    y = np.empty((T, H), np.float64)
    rc = lib.oracle_bruteforce(_p(xa), ctypes.c_int32(xdt), ctypes.c_int64(T), ctypes.c_int32(H), _p(lg),
                               ctypes.c_int32(ldt), ctypes.c_int32(E), ctypes.c_int32(k), ctypes.c_int32(D),
                               ctypes.c_int32(d), _p(ga), _p(ua), _p(da), ctypes.c_int32(wdt), _p(nidx),
                               ctypes.c_int32(0 if act == "swiglu" else 1), _p(y))
    _check(rc, "oracle_bruteforce")
    return y


def ep_sim(G: int, x, logits, k: int, w_gate, w_up, w_down, act: str = "swiglu",
           nthreads: int | None = None):
    """Expert-parallel layer simulated in one address space over G ranks."""
    lib = _load()
    xa, xdt = _as_input(x)
    lg, ldt = _as_input(logits)
    (wg, wu, wd), wdt = _weights(w_gate, w_up, w_down)
    T, H = xa.shape
    E, d, _H = wg.shape
    y = np.empty((T, H), np.float64)
    rc = lib.oracle_ep_sim(ctypes.c_int32(G), _p(xa), ctypes.c_int32(xdt), ctypes.c_int64(T),
                           ctypes.c_int32(H), _p(lg), ctypes.c_int32(ldt), ctypes.c_int32(E),
                           ctypes.c_int32(k), ctypes.c_int32(d), _p(wg), _p(wu), _p(wd),
                           ctypes.c_int32(wdt), ctypes.c_int32(0 if act == "swiglu" else 1), _p(y),
                           ctypes.c_int32(nthreads or default_threads()))
    _check(rc, "oracle_ep_sim")
    return y
