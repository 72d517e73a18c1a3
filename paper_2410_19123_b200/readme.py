"""Thin Python binding over libreadme_b200.so (include/readme.h). Argument marshalling only: every step
of the path runs in the library's CUDA kernels; PyTorch supplies device memory and streams.

There is no CPU fallback: if the library is missing, or a tensor is not on a CUDA device, the call
raises. Names follow the C ABI (route, dispatch, expert_ffn, combine, moe_layer, build_experts).
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libreadme_b200.so")

README_F32, README_BF16 = 0, 1
README_DEV_NONFINITE_LOGIT, README_DEV_BAD_INDEX = 0x1, 0x2
README_DEV_SCHED_TIMEOUT, README_DEV_EP_TIMEOUT = 0x4, 0x8  # include/readme.h
STATUS = {0: "README_OK", 1: "README_ERR_INVALID_ARG", 2: "README_ERR_UNSUPPORTED", 3: "README_ERR_WORKSPACE",
          4: "README_ERR_CUDA"}

# Every symbol include/readme.h declares (tests check the library exports exactly these).
EXPORTS = ("readme_route_workspace_bytes", "readme_route", "readme_dispatch", "readme_expert_ffn_workspace_bytes",
           "readme_expert_ffn", "readme_expert_gate_up", "readme_expert_down", "readme_combine", "readme_moe_layer_workspace_bytes", "readme_moe_layer",
           "readme_build_experts", "readme_permanent_expert_workspace_bytes", "readme_permanent_expert",
           "readme_router_workspace_bytes", "readme_router_forward", "readme_router_step_workspace_bytes",
           "readme_router_step", "readme_router_route_workspace_bytes", "readme_router_forward_route",
           "readme_dispatch_rmsnorm", "readme_moe_stack_workspace_bytes", "readme_moe_stack",
           "readme_scheduler_create", "readme_scheduler_destroy", "readme_scheduler_push", "readme_scheduler_queued",
           "readme_scheduler_next_batch", "readme_expert_ffn_slots", "readme_cache_create", "readme_cache_destroy",
           "readme_cache_set_future", "readme_cache_access", "readme_cache_lookup", "readme_cache_stats",
           "readme_ep_alloc", "readme_ep_free", "readme_ipc_handle", "readme_ipc_open", "readme_ipc_close",
           "readme_ep_signal", "readme_ep_wait", "readme_ep_publish_counts", "readme_ep_plan", "readme_ep_dispatch",
           "readme_ep_expert_ffn",
           "readme_set_device", "readme_status_string", "readme_last_error",
           "readme_version", "readme_debug_trace", "readme_debug_tile_trace", "readme_debug_mark", "readme_debug_set_knob",
           "readme_debug_get_knob", "readme_debug_reset_knob", "readme_debug_hold_sms")


class ReadmeError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None
_lock = threading.Lock()
_tls = threading.local()

_vp, _i32, _i64, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_SIGS = {
    "readme_route_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "readme_route": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                                    _vp]),
    "readme_dispatch": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _vp, _vp, _vp, _vp]),
    "readme_expert_ffn_workspace_bytes": (_sz, [_i64, _i32, _i32, _i32, ctypes.c_int]),
    "readme_expert_ffn": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                         _vp, _vp, _sz, _vp]),
    "readme_expert_gate_up": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp,
                                             _vp]),
    "readme_expert_down": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                          _vp]),
    "readme_combine": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "readme_moe_layer_workspace_bytes": (_sz, [_i64, _i32, _i32, _i32, _i32, ctypes.c_int]),
    "readme_moe_layer": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _vp, ctypes.c_int, _i32, _i32, _i32, _vp, _vp,
                                        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "readme_build_experts": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp,
                                            _vp, _vp]),
    "readme_dispatch_rmsnorm": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _vp, ctypes.c_float, _vp, _vp,
                                               _vp]),
    "readme_moe_stack_workspace_bytes": (_sz, [_i64, _i32, _i32, _i32, _i32, ctypes.c_int]),
    "readme_moe_stack": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _vp, ctypes.c_int, _i32, _i32, _i32, _i32,
                                        _vp, _vp, _vp, ctypes.c_float, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                                        _vp]),
    "readme_scheduler_create": (_vp, [_i32]),
    "readme_scheduler_destroy": (None, [_vp]),
    "readme_scheduler_push": (ctypes.c_int, [_vp, _vp, _vp, _i64]),
    "readme_scheduler_queued": (_i64, [_vp, _i32]),
    "readme_scheduler_next_batch": (_i64, [_vp, _i64, _vp, _vp]),
    "readme_permanent_expert_workspace_bytes": (_sz, [_i64, _i32, _i32, ctypes.c_int]),
    "readme_permanent_expert": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp,
                                               _sz, _vp]),
    "readme_router_workspace_bytes": (_sz, [_i64, _i32]),
    "readme_router_step_workspace_bytes": (_sz, [_i64, _i32]),
    "readme_router_step": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _i32, _i32, _vp, ctypes.c_float, _vp, _vp, _vp,
                                          _sz, _vp]),
    "readme_router_forward": (ctypes.c_int, [_vp, _i64, _vp, _i32, _vp, ctypes.c_float, _vp, _vp, _vp, _sz, _vp]),
    "readme_router_route_workspace_bytes": (_sz, [_i64, _i32, _i32, _i32]),
    "readme_router_forward_route": (ctypes.c_int, [_vp, _i64, _vp, _i32, _vp, ctypes.c_float, _i32, _vp, _vp, _vp,
                                                   _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "readme_expert_ffn_slots": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _i32, _vp, _vp, _i32, _vp, _vp,
                                               _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "readme_cache_create": (_vp, [_i32, _i32, ctypes.c_uint64]),
    "readme_cache_destroy": (None, [_vp]),
    "readme_cache_set_future": (ctypes.c_int, [_vp, _vp, _vp, _i64]),
    "readme_cache_access": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "readme_cache_lookup": (_i32, [_vp, _i64]),
    "readme_cache_stats": (None, [_vp, _vp, _vp]),
    "readme_ep_alloc": (ctypes.c_int, [_sz, _vp]),
    "readme_ep_free": (ctypes.c_int, [_vp]),
    "readme_ipc_handle": (ctypes.c_int, [_vp, _vp]),
    "readme_ipc_open": (ctypes.c_int, [_vp, _vp]),
    "readme_ipc_close": (ctypes.c_int, [_vp]),
    "readme_ep_signal": (ctypes.c_int, [_vp, _i32, _i32, _vp, _vp]),
    "readme_ep_wait": (ctypes.c_int, [_vp, _i32, _vp, _vp, _vp]),
    "readme_ep_publish_counts": (ctypes.c_int, [_vp, _i32, _vp, _i32, _i32, _vp]),
    "readme_ep_plan": (ctypes.c_int, [_vp, _i32, _i32, _i32, _vp, _vp, _vp]),
    "readme_ep_dispatch": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _vp, _vp, _vp, _i32, _i32, _i32, _vp,
                                          _vp, _i64, _i32, _vp, _vp]),
    "readme_ep_expert_ffn": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                            _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "readme_set_device": (ctypes.c_int, [ctypes.c_int]),
    "readme_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "readme_last_error": (ctypes.c_char_p, []),
    "readme_version": (ctypes.c_int, []),
    "readme_debug_trace": (None, [_vp]),
    "readme_debug_tile_trace": (None, [_vp, _i32]),
    "readme_debug_mark": (ctypes.c_int, [_i32, _vp]),
    "readme_debug_set_knob": (ctypes.c_int, [ctypes.c_char_p, _i32]),
    "readme_debug_get_knob": (ctypes.c_int, [ctypes.c_char_p, _vp]),
    "readme_debug_reset_knob": (ctypes.c_int, [ctypes.c_char_p]),
    "readme_debug_hold_sms": (ctypes.c_int, [_i32, _i64, _vp]),
}


def lib():
    """Load libreadme_b200.so (raises if it is missing: there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2410_19123_b200.build` "
                                  "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_LOCAL)
            for name, (res, args) in _SIGS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _check(fn: str, rc: int):
    if rc != 0:
        raise ReadmeError(fn, rc, lib().readme_last_error().decode(errors="replace"))


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return README_BF16
    if t.dtype == torch.float32:
        return README_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or f32)")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _prep(*tensors):
    """All tensors must be contiguous CUDA tensors on one device; binds the library's thread to it and
    returns the current torch stream handle."""
    dev = None
    for t in tensors:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("readme: tensors must live on a CUDA device (no CPU path exists)")
        if not t.is_contiguous():
            raise ValueError("readme: tensors must be contiguous")
        if dev is None:
            dev = t.device.index
        elif t.device.index != dev:
            raise ValueError("readme: tensors on different devices")
    if dev is None:
        dev = torch.cuda.current_device()
    if getattr(_tls, "dev", None) != dev:
        _check("readme_set_device", lib().readme_set_device(dev))
        _tls.dev = dev
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


@dataclass
class Plan:
    """The routing plan (a1-a4): computed once per batch, reused by every layer (a9)."""
    topk_idx: torch.Tensor   # [T,k] int32
    topk_w: torch.Tensor     # [T,k] f32
    counts: torch.Tensor     # [E] int32
    offsets: torch.Tensor    # [E+1] int32
    dest: torch.Tensor       # [T*k] int32
    src: torch.Tensor        # [T*k] int32
    dev_status: torch.Tensor  # [1] int32 (uint32 bits)

    @property
    def k(self) -> int:
        return self.topk_idx.shape[1]


def new_plan(T: int, E: int, k: int, device) -> Plan:
    i32 = dict(dtype=torch.int32, device=device)
    return Plan(torch.empty((T, k), **i32), torch.empty((T, k), dtype=torch.float32, device=device),
                torch.empty(E, **i32), torch.empty(E + 1, **i32), torch.empty(T * k, **i32),
                torch.empty(T * k, **i32), torch.zeros(1, **i32))


def route_workspace_bytes(T: int, E: int, k: int) -> int:
    return int(lib().readme_route_workspace_bytes(T, E, k))


def route(logits: torch.Tensor, k: int, plan: Plan | None = None, ws: torch.Tensor | None = None) -> Plan:
    """a1-a4 on the device: top-k ids/weights, counts, offsets, dest, src (readme_route)."""
    T, E = logits.shape
    plan = plan or new_plan(T, E, k, logits.device)
    need = route_workspace_bytes(T, E, k)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=logits.device)
    st = _prep(logits, plan.topk_idx, ws)
    _check("readme_route", lib().readme_route(
        _ptr(logits), _dt(logits), T, E, k, _ptr(plan.topk_idx), _ptr(plan.topk_w), _ptr(plan.counts),
        _ptr(plan.offsets), _ptr(plan.dest), _ptr(plan.src), _ptr(plan.dev_status), _ptr(ws), ws.numel(), st))
    return plan


def dispatch(x: torch.Tensor, dest: torch.Tensor, k: int, out: torch.Tensor | None = None,
             dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """a5: x_sorted[dest[s]] = x[s // k] (readme_dispatch)."""
    T, H = x.shape
    out = out if out is not None else torch.empty((T * k, H), dtype=x.dtype, device=x.device)
    st = _prep(x, dest, out, dev_status)
    _check("readme_dispatch", lib().readme_dispatch(_ptr(x), _dt(x), T, H, k, _ptr(dest), _ptr(out),
                                                    _ptr(dev_status), st))
    return out


def expert_ffn_workspace_bytes(rows: int, H: int, E: int, d: int, dtype: torch.dtype) -> int:
    return int(lib().readme_expert_ffn_workspace_bytes(rows, H, E, d,
                                                       README_BF16 if dtype == torch.bfloat16 else README_F32))


def expert_ffn(x_sorted: torch.Tensor, offsets: torch.Tensor, w_gate: torch.Tensor, w_up: torch.Tensor,
               w_down: torch.Tensor, n_src: int = 1, out: torch.Tensor | None = None,
               ws: torch.Tensor | None = None, dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """a6-a7: grouped SwiGLU expert FFN over expert-contiguous rows (readme_expert_ffn). dev_status: optional
    uint32/int32 device word that README_DEV_SCHED_TIMEOUT is OR-ed into."""
    rows, H = x_sorted.shape
    E, d, H2 = w_gate.shape
    if H2 != H or tuple(w_up.shape) != (E, d, H) or tuple(w_down.shape) != (E, H, d):
        raise ValueError("weight shapes must be w_gate/w_up [E,d,H] and w_down [E,H,d]")
    if not (x_sorted.dtype == w_gate.dtype == w_up.dtype == w_down.dtype):
        raise TypeError("x_sorted and weights must share a dtype")
    out = out if out is not None else torch.empty((rows, H), dtype=x_sorted.dtype, device=x_sorted.device)
    need = expert_ffn_workspace_bytes(rows, H, E, d, x_sorted.dtype)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=x_sorted.device)
    st = _prep(x_sorted, offsets, w_gate, w_up, w_down, out, ws)
    _check("readme_expert_ffn", lib().readme_expert_ffn(
        _ptr(x_sorted), _dt(x_sorted), rows, H, E, d, n_src, _ptr(offsets), _ptr(w_gate), _ptr(w_up),
        _ptr(w_down), _ptr(out), _ptr(dev_status), _ptr(ws), ws.numel(), st))
    return out


def expert_gate_up(x_sorted: torch.Tensor, offsets: torch.Tensor, w_gate: torch.Tensor, w_up: torch.Tensor,
                   n_src: int = 1, out: torch.Tensor | None = None) -> torch.Tensor:
    """a6: h = silu(x_sorted W_gate[e]^T) * (x_sorted W_up[e]^T) per segment (readme_expert_gate_up)."""
    rows, H = x_sorted.shape
    E, d, _ = w_gate.shape
    out = out if out is not None else torch.empty((rows, d), dtype=x_sorted.dtype, device=x_sorted.device)
    st = _prep(x_sorted, offsets, w_gate, w_up, out)
    _check("readme_expert_gate_up", lib().readme_expert_gate_up(
        _ptr(x_sorted), _dt(x_sorted), rows, H, E, d, n_src, _ptr(offsets), _ptr(w_gate), _ptr(w_up), _ptr(out), st))
    return out


def expert_down(h: torch.Tensor, offsets: torch.Tensor, w_down: torch.Tensor, n_src: int = 1,
                src: torch.Tensor | None = None, residual: torch.Tensor | None = None,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """a7: y_sorted = h W_down[e]^T per segment; with src (k == 1) rows go to out[src[r]] + residual, i.e. the
    combine fused into the epilogue (readme_expert_down)."""
    rows, d = h.shape
    E, H, _ = w_down.shape
    out = out if out is not None else torch.empty((rows, H), dtype=h.dtype, device=h.device)
    st = _prep(h, offsets, w_down, src, residual, out)
    _check("readme_expert_down", lib().readme_expert_down(
        _ptr(h), _dt(h), rows, H, E, d, n_src, _ptr(offsets), _ptr(w_down), _ptr(src), _ptr(residual), _ptr(out),
        st))
    return out


def combine(y_sorted: torch.Tensor, dest: torch.Tensor, topk_w: torch.Tensor | None, k: int,
            residual: torch.Tensor | None = None, out: torch.Tensor | None = None,
            dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """a8: y[t] = residual[t] + sum_j w[t,j] * y_sorted[dest[t*k+j]] (readme_combine)."""
    rows, H = y_sorted.shape
    T = rows // k
    out = out if out is not None else torch.empty((T, H), dtype=y_sorted.dtype, device=y_sorted.device)
    st = _prep(y_sorted, dest, topk_w, residual, out, dev_status)
    _check("readme_combine", lib().readme_combine(_ptr(y_sorted), _dt(y_sorted), T, H, k, _ptr(dest), _ptr(topk_w),
                                                  _ptr(residual), _ptr(out), _ptr(dev_status), st))
    return out


def moe_layer_workspace_bytes(T: int, H: int, E: int, d: int, k: int, dtype: torch.dtype) -> int:
    return int(lib().readme_moe_layer_workspace_bytes(T, H, E, d, k,
                                                      README_BF16 if dtype == torch.bfloat16 else README_F32))


def moe_layer(x: torch.Tensor, w_gate: torch.Tensor, w_up: torch.Tensor, w_down: torch.Tensor, k: int = 1,
              logits: torch.Tensor | None = None, plan: Plan | None = None, residual: torch.Tensor | None = None,
              out: torch.Tensor | None = None, ws: torch.Tensor | None = None) -> tuple[torch.Tensor, Plan]:
    """The whole layer (readme_moe_layer). With `logits` the plan is computed (into `plan` if given);
    with logits=None, `plan` is an input (route once, reuse for every layer)."""
    T, H = x.shape
    E, d, _ = w_gate.shape
    if logits is None and plan is None:
        raise ValueError("moe_layer needs logits or a plan")
    if plan is None:
        plan = new_plan(T, E, k, x.device)
    k = plan.k
    out = out if out is not None else torch.empty_like(x)
    need = moe_layer_workspace_bytes(T, H, E, d, k, x.dtype)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=x.device)
    st = _prep(x, w_gate, w_up, w_down, logits, residual, out, ws, plan.dest)
    _check("readme_moe_layer", lib().readme_moe_layer(
        _ptr(x), _dt(x), T, H, _ptr(logits), _dt(logits) if logits is not None else README_F32, E, k, d,
        _ptr(w_gate), _ptr(w_up), _ptr(w_down), _ptr(residual), _ptr(out), _ptr(plan.topk_idx),
        _ptr(plan.topk_w), _ptr(plan.counts), _ptr(plan.offsets), _ptr(plan.dest), _ptr(plan.src),
        _ptr(plan.dev_status), _ptr(ws), ws.numel(), st))
    return out, plan


def build_experts(dense_w_gate: torch.Tensor, dense_w_up: torch.Tensor, dense_w_down: torch.Tensor,
                  neuron_idx: torch.Tensor, dev_status: torch.Tensor | None = None):
    """Setup: slice expert stacks from the dense FFN (readme_build_experts). Returns (w_gate, w_up, w_down)."""
    D, H = dense_w_gate.shape
    E, d = neuron_idx.shape
    kw = dict(dtype=dense_w_gate.dtype, device=dense_w_gate.device)
    wg = torch.empty((E, d, H), **kw)
    wu = torch.empty((E, d, H), **kw)
    wd = torch.empty((E, H, d), **kw)
    st = _prep(dense_w_gate, dense_w_up, dense_w_down, neuron_idx, wg, wu, wd, dev_status)
    _check("readme_build_experts", lib().readme_build_experts(
        _ptr(dense_w_gate), _ptr(dense_w_up), _ptr(dense_w_down), _dt(dense_w_gate), D, H, E, d, _ptr(neuron_idx),
        _ptr(wg), _ptr(wu), _ptr(wd), _ptr(dev_status), st))
    return wg, wu, wd


def dispatch_rmsnorm(x: torch.Tensor, dest: torch.Tensor, k: int, eps: float = 1e-5, out: torch.Tensor | None = None,
                     dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """Pre-norm dispatch: x_sorted[dest[t*k+j]] = RMSNorm(x[t]) (readme_dispatch_rmsnorm)."""
    T, H = x.shape
    out = out if out is not None else torch.empty((T * k, H), dtype=x.dtype, device=x.device)
    st = _prep(x, dest, out, dev_status)
    _check("readme_dispatch_rmsnorm", lib().readme_dispatch_rmsnorm(_ptr(x), _dt(x), T, H, k, _ptr(dest),
                                                                    ctypes.c_float(eps), _ptr(out), _ptr(dev_status),
                                                                    st))
    return out


def moe_stack_workspace_bytes(T: int, H: int, E: int, d: int, k: int, dtype: torch.dtype) -> int:
    return int(lib().readme_moe_stack_workspace_bytes(T, H, E, d, k,
                                                      README_BF16 if dtype == torch.bfloat16 else README_F32))


def moe_stack(x: torch.Tensor, layers, k: int = 1, logits: torch.Tensor | None = None, plan: Plan | None = None,
              eps: float = 1e-5, ws: torch.Tensor | None = None) -> tuple[torch.Tensor, Plan]:
    """L pre-norm MoE layers routed once (readme_moe_stack). `layers` = [(w_gate, w_up, w_down), ...];
    x is updated in place and returned."""
    T, H = x.shape
    L = len(layers)
    E, d, _ = layers[0][0].shape if L else (0, 8, 0)
    if logits is None and plan is None:
        raise ValueError("moe_stack needs logits or a plan")
    if plan is None:
        plan = new_plan(T, logits.shape[1], k, x.device)
        E = logits.shape[1]
    k = plan.k
    need = moe_stack_workspace_bytes(T, H, E, d, k, x.dtype)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=x.device)
    arr = ctypes.c_void_p * max(L, 1)
    wg = arr(*[w[0].data_ptr() for w in layers])
    wu = arr(*[w[1].data_ptr() for w in layers])
    wd = arr(*[w[2].data_ptr() for w in layers])
    st = _prep(x, logits, ws, plan.dest, *[t for w in layers for t in w])
    _check("readme_moe_stack", lib().readme_moe_stack(
        _ptr(x), _dt(x), T, H, _ptr(logits), _dt(logits) if logits is not None else README_F32, E, k, d, L,
        ctypes.cast(wg, ctypes.c_void_p), ctypes.cast(wu, ctypes.c_void_p), ctypes.cast(wd, ctypes.c_void_p),
        ctypes.c_float(eps), _ptr(plan.topk_idx), _ptr(plan.topk_w), _ptr(plan.counts), _ptr(plan.offsets),
        _ptr(plan.dest), _ptr(plan.src), _ptr(plan.dev_status), _ptr(ws), ws.numel(), st))
    return x, plan


class ExpertScheduler:
    """Expert-aware batching (Alg. 1) over per-expert FIFO queues, in the native host
    runtime (readme_scheduler_*)."""

    def __init__(self, E: int):
        import numpy as np
        self._np = np
        self.E = E
        self._h = lib().readme_scheduler_create(E)
        if not self._h:
            raise ValueError(f"readme_scheduler_create({E}) failed")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().readme_scheduler_destroy(h)
            self._h = None

    def push(self, token_ids, experts):
        np = self._np
        t = np.ascontiguousarray(token_ids, dtype=np.int64)
        e = np.ascontiguousarray(experts, dtype=np.int32)
        if t.shape != e.shape:
            raise ValueError("token_ids and experts must have the same length")
        _check("readme_scheduler_push", lib().readme_scheduler_push(
            self._h, t.ctypes.data_as(ctypes.c_void_p), e.ctypes.data_as(ctypes.c_void_p), t.size))

    def queued(self, e: int = -1) -> int:
        return int(lib().readme_scheduler_queued(self._h, e))

    def next_batch(self, max_tokens: int):
        """Returns (token_ids int64 [n], experts int32 [n]) of the next batch (grouped by expert)."""
        np = self._np
        t = np.empty(max(max_tokens, 1), np.int64)
        e = np.empty(max(max_tokens, 1), np.int32)
        n = lib().readme_scheduler_next_batch(self._h, max_tokens, t.ctypes.data_as(ctypes.c_void_p),
                                              e.ctypes.data_as(ctypes.c_void_p))
        if n < 0:
            raise ValueError("readme_scheduler_next_batch: bad argument")
        return t[:n].copy(), e[:n].copy()


def permanent_expert(x: torch.Tensor, w_gate: torch.Tensor, w_up: torch.Tensor, w_down: torch.Tensor,
                     y: torch.Tensor, ws: torch.Tensor | None = None,
                     dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """y += F_perm(x) for every token (the permanent expert; readme_permanent_expert)."""
    T, H = x.shape
    dp = w_gate.shape[0]
    need = int(lib().readme_permanent_expert_workspace_bytes(T, H, dp, _dt(x)))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=x.device)
    st = _prep(x, w_gate, w_up, w_down, y, ws)
    _check("readme_permanent_expert", lib().readme_permanent_expert(
        _ptr(x), _dt(x), T, H, dp, _ptr(w_gate), _ptr(w_up), _ptr(w_down), _ptr(y),
        _ptr(dev_status), _ptr(ws), ws.numel(), st))
    return y


class _RouterWeights(ctypes.Structure):
    _fields_ = [("vocab", ctypes.c_int32), ("n_experts", ctypes.c_int32)] + \
               [(n, ctypes.c_void_p) for n in ("emb", "norm1", "w_qkv", "w_o", "norm2", "w_gate", "w_up", "w_down",
                                               "norm_f", "w_head")]


ROUTER_KEYS = ("emb", "norm1", "w_qkv", "w_o", "norm2", "w_gate", "w_up", "w_down", "norm_f", "w_head")


def router_workspace_bytes(T: int, nseq: int) -> int:
    return int(lib().readme_router_workspace_bytes(T, nseq))


def router_forward(token_ids: torch.Tensor, seq_starts: torch.Tensor, weights: dict, eps: float = 1e-5,
                   out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                   dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """The pre-gating router G: token ids -> expert logits [T, N] f32 (readme_router_forward). `weights` maps
    ROUTER_KEYS to bf16 CUDA tensors (nn.Linear [out, in] layouts)."""
    T = token_ids.numel()
    nseq = seq_starts.numel() - 1
    N = weights["w_head"].shape[0]
    out = out if out is not None else torch.empty((T, N), dtype=torch.float32, device=token_ids.device)
    need = int(lib().readme_router_workspace_bytes(T, nseq))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=token_ids.device)
    st = _prep(token_ids, seq_starts, out, ws, dev_status, *[weights[k] for k in ROUTER_KEYS])
    w = _RouterWeights(weights["emb"].shape[0], N, *[weights[k].data_ptr() for k in ROUTER_KEYS])
    _check("readme_router_forward", lib().readme_router_forward(
        _ptr(token_ids), T, _ptr(seq_starts), nseq, ctypes.cast(ctypes.pointer(w), ctypes.c_void_p),
        ctypes.c_float(eps), _ptr(out), _ptr(dev_status), _ptr(ws), ws.numel(), st))
    return out


def router_forward_route(token_ids: torch.Tensor, seq_starts: torch.Tensor, weights: dict, k: int = 1,
                         eps: float = 1e-5, plan: Plan | None = None, out: torch.Tensor | None = None,
                         ws: torch.Tensor | None = None) -> tuple[torch.Tensor, Plan]:
    """The router and the routing plan in one call (readme_router_forward_route): the block, then ONE route
    launch that computes the final RMSNorm + gating head + a1-a4 from the block's hidden state. Returns
    (logits [T, N] f32, plan)."""
    T = token_ids.numel()
    nseq = seq_starts.numel() - 1
    N = weights["w_head"].shape[0]
    dev = token_ids.device
    out = out if out is not None else torch.empty((T, N), dtype=torch.float32, device=dev)
    plan = plan if plan is not None else new_plan(T, N, k, dev)
    need = int(lib().readme_router_route_workspace_bytes(T, nseq, N, k))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
    st = _prep(token_ids, seq_starts, out, ws, *[weights[kk] for kk in ROUTER_KEYS], *plan_tensors(plan))
    w = _RouterWeights(weights["emb"].shape[0], N, *[weights[kk].data_ptr() for kk in ROUTER_KEYS])
    _check("readme_router_forward_route", lib().readme_router_forward_route(
        _ptr(token_ids), T, _ptr(seq_starts), nseq, ctypes.cast(ctypes.pointer(w), ctypes.c_void_p),
        ctypes.c_float(eps), k, _ptr(out), _ptr(plan.topk_idx), _ptr(plan.topk_w), _ptr(plan.counts),
        _ptr(plan.offsets), _ptr(plan.dest), _ptr(plan.src), _ptr(plan.dev_status), _ptr(ws), ws.numel(), st))
    return out, plan


def plan_tensors(plan: Plan):
    return (plan.topk_idx, plan.topk_w, plan.counts, plan.offsets, plan.dest, plan.src, plan.dev_status)


def new_router_cache(n_slots: int, max_len: int, device) -> torch.Tensor:
    """Key/value cache for readme_router_step: bf16 [n_slots, max_len, 2, 512]."""
    return torch.zeros((n_slots, max_len, 2, 512), dtype=torch.bfloat16, device=device)


def router_step(token_ids: torch.Tensor, slot: torch.Tensor, pos: torch.Tensor, kv_cache: torch.Tensor,
                weights: dict, eps: float = 1e-5, out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """Incremental router (readme_router_step): new tokens (request slot, position) -> logits [n, N] f32; their
    keys/values are appended to kv_cache."""
    n = token_ids.numel()
    N = weights["w_head"].shape[0]
    n_slots, max_len = kv_cache.shape[0], kv_cache.shape[1]
    out = out if out is not None else torch.empty((n, N), dtype=torch.float32, device=token_ids.device)
    need = int(lib().readme_router_step_workspace_bytes(n, max_len))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=token_ids.device)
    st = _prep(token_ids, slot, pos, kv_cache, out, ws, dev_status, *[weights[k] for k in ROUTER_KEYS])
    w = _RouterWeights(weights["emb"].shape[0], N, *[weights[k].data_ptr() for k in ROUTER_KEYS])
    _check("readme_router_step", lib().readme_router_step(
        _ptr(token_ids), n, _ptr(slot), _ptr(pos), _ptr(kv_cache), n_slots, max_len,
        ctypes.cast(ctypes.pointer(w), ctypes.c_void_p), ctypes.c_float(eps), _ptr(out), _ptr(dev_status), _ptr(ws),
        ws.numel(), st))
    return out


def expert_ffn_slots(x_sorted: torch.Tensor, offsets: torch.Tensor, expert_slot: torch.Tensor, w_gate: torch.Tensor,
                     w_up: torch.Tensor, w_down: torch.Tensor, E: int, src: torch.Tensor | None = None,
                     residual: torch.Tensor | None = None, out: torch.Tensor | None = None,
                     ws: torch.Tensor | None = None, dev_status: torch.Tensor | None = None) -> torch.Tensor:
    """Expert FFN over slot pools (readme_expert_ffn_slots): expert e's weights at slot expert_slot[e]."""
    rows, H = x_sorted.shape
    S, d, _ = w_gate.shape
    if out is None:
        out = torch.empty((rows, H), dtype=x_sorted.dtype, device=x_sorted.device)
    need = expert_ffn_workspace_bytes(rows, H, E, d, x_sorted.dtype)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=x_sorted.device)
    st = _prep(x_sorted, offsets, expert_slot, w_gate, w_up, w_down, src, residual, out, ws, dev_status)
    _check("readme_expert_ffn_slots", lib().readme_expert_ffn_slots(
        _ptr(x_sorted), _dt(x_sorted), rows, H, E, d, _ptr(offsets), _ptr(expert_slot), S, _ptr(w_gate),
        _ptr(w_up), _ptr(w_down), _ptr(src), _ptr(residual), _ptr(out), _ptr(dev_status), _ptr(ws), ws.numel(), st))
    return out


class ExpertCache:
    """Expert cache policy in the native runtime (readme_cache_*): LRU, Belady (pre-gated future), Random."""
    POLICIES = {"lru": 0, "belady": 1, "random": 2}

    def __init__(self, capacity: int, policy: str, seed: int = 0):
        self._h = lib().readme_cache_create(capacity, self.POLICIES[policy], seed)
        if not self._h:
            raise ValueError("readme_cache_create failed")
        self.capacity = capacity

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().readme_cache_destroy(h)
            self._h = None

    def set_future(self, keys, times):
        import numpy as np
        k = np.ascontiguousarray(keys, dtype=np.int64)
        t = np.ascontiguousarray(times, dtype=np.int64)
        _check("readme_cache_set_future", lib().readme_cache_set_future(
            self._h, k.ctypes.data_as(ctypes.c_void_p), t.ctypes.data_as(ctypes.c_void_p), k.size))

    def access(self, key: int, t: int, protect_since: int = 2 ** 63 - 1):
        """Returns (hit: bool, slot: int, evicted: int or -1). Residents accessed at or after protect_since are
        not evictable."""
        ev = ctypes.c_int64(-1)
        sl = ctypes.c_int32(-1)
        r = lib().readme_cache_access(self._h, key, t, protect_since, ctypes.byref(ev), ctypes.byref(sl))
        if r == -2:
            raise RuntimeError("expert cache full of protected experts: capacity below one layer's working set")
        if r < 0:
            raise ValueError("readme_cache_access: bad argument")
        return bool(r), int(sl.value), int(ev.value)

    def lookup(self, key: int) -> int:
        return int(lib().readme_cache_lookup(self._h, key))

    def stats(self):
        h, m = ctypes.c_int64(0), ctypes.c_int64(0)
        lib().readme_cache_stats(self._h, ctypes.byref(h), ctypes.byref(m))
        return int(h.value), int(m.value)


# ---- expert parallelism over peer memory (readme_ep_*, readme_ipc_*) ----------------------------------

IPC_HANDLE_BYTES = 64


def _ptrs(v):
    """Host array of device pointers (ints) for the peer_* arguments."""
    return (ctypes.c_void_p * len(v))(*[None if p is None else int(p) for p in v])


def _stream_for(device=None):
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    if getattr(_tls, "dev", None) != dev:
        _check("readme_set_device", lib().readme_set_device(dev))
        _tls.dev = dev
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def ep_alloc(nbytes: int, device=None) -> int:
    """Zero-filled device memory owned by the library (IPC-exportable); returns the device pointer."""
    _stream_for(device)
    p = ctypes.c_void_p()
    _check("readme_ep_alloc", lib().readme_ep_alloc(nbytes, ctypes.byref(p)))
    return int(p.value)


def ep_free(ptr: int):
    _check("readme_ep_free", lib().readme_ep_free(ctypes.c_void_p(ptr)))


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check("readme_ipc_handle", lib().readme_ipc_handle(ctypes.c_void_p(ptr), buf))
    return buf.raw


def ipc_open(handle: bytes, device=None) -> int:
    _stream_for(device)
    p = ctypes.c_void_p()
    _check("readme_ipc_open", lib().readme_ipc_open(ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES),
                                                    ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int):
    _check("readme_ipc_close", lib().readme_ipc_close(ctypes.c_void_p(ptr)))


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


_TYPESTR = {torch.bfloat16: "<V2", torch.int32: "<i4", torch.int64: "<i8", torch.float32: "<f4",
            torch.uint8: "|u1"}


def device_view(ptr: int, shape, dtype, device) -> torch.Tensor:
    """A torch tensor over library-owned device memory (no copy)."""
    if dtype == torch.bfloat16:  # no bf16 typestr in the interface: view int16 storage as bf16
        return torch.as_tensor(_CAI(ptr, shape, "<i2"), device=device).view(torch.bfloat16)
    return torch.as_tensor(_CAI(ptr, shape, _TYPESTR[dtype]), device=device)


def ep_signal(peer_flags, me: int, epoch: int, device=None):
    """epoch: device pointer to this rank's uint64 phase counter."""
    st = _stream_for(device)
    _check("readme_ep_signal", lib().readme_ep_signal(_ptrs(peer_flags), len(peer_flags), me,
                                                      ctypes.c_void_p(epoch), st))


def ep_wait(flags: int, G: int, epoch: int, dev_status: torch.Tensor | None = None, device=None):
    st = _stream_for(device)
    _check("readme_ep_wait", lib().readme_ep_wait(ctypes.c_void_p(flags), G, ctypes.c_void_p(epoch),
                                                  _ptr(dev_status), st))


def ep_publish_counts(counts: torch.Tensor, peer_tables, me: int):
    st = _prep(counts)
    _check("readme_ep_publish_counts", lib().readme_ep_publish_counts(_ptr(counts), counts.numel(),
                                                                      _ptrs(peer_tables), len(peer_tables), me, st))


def ep_plan(table: int, G: int, E: int, me: int, seg_offsets: torch.Tensor, row_base: torch.Tensor):
    st = _prep(seg_offsets, row_base)
    _check("readme_ep_plan", lib().readme_ep_plan(ctypes.c_void_p(table), G, E, me, _ptr(seg_offsets),
                                                  _ptr(row_base), st))


def ep_dispatch(x: torch.Tensor, k: int, dest, offsets, row_base, E: int, me: int, peer_x, peer_map, vrows: int,
                to_token: bool, dev_status: torch.Tensor | None = None):
    st = _prep(x, dest, offsets, row_base, dev_status)
    T, H = x.shape
    _check("readme_ep_dispatch", lib().readme_ep_dispatch(
        _ptr(x), _dt(x), T, H, k, _ptr(dest), _ptr(offsets), _ptr(row_base), E, len(peer_x), me, _ptrs(peer_x),
        _ptrs(peer_map), vrows, int(bool(to_token)), _ptr(dev_status), st))


def ep_expert_ffn(x_recv: torch.Tensor, seg_offsets, w_gate, w_up, w_down, row_map, peer_out, peer_res, vrows: int,
                  ws: torch.Tensor, dev_status: torch.Tensor | None = None):
    st = _prep(x_recv, seg_offsets, w_gate, w_up, w_down, row_map, ws, dev_status)
    rows_cap, H = x_recv.shape
    El, d, _ = w_gate.shape
    G = len(peer_out)
    res = _ptrs(peer_res) if peer_res is not None else None
    _check("readme_ep_expert_ffn", lib().readme_ep_expert_ffn(
        _ptr(x_recv), _dt(x_recv), rows_cap, H, El, d, G, _ptr(seg_offsets), _ptr(w_gate), _ptr(w_up),
        _ptr(w_down), _ptr(row_map), _ptrs(peer_out), res, vrows, _ptr(dev_status), _ptr(ws), ws.numel(), st))


# ---- lab / test switches (readme_debug_set_knob) ---------------------------------------------

def set_knob(name: str, value: int) -> None:
    _check("readme_debug_set_knob", lib().readme_debug_set_knob(name.encode(), int(value)))


def get_knob(name: str) -> int:
    v = ctypes.c_int32(0)
    _check("readme_debug_get_knob", lib().readme_debug_get_knob(name.encode(), ctypes.byref(v)))
    return int(v.value)


def reset_knob(name: str) -> None:
    _check("readme_debug_reset_knob", lib().readme_debug_reset_knob(name.encode()))


class knobs:
    """Context manager: `with rd.knobs(ffn_mt=128, route=2): ...` sets the switches, restores them after."""

    def __init__(self, **kv):
        self.kv = kv
        self.old = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.old[k] = get_knob(k)
            set_knob(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            set_knob(k, v)


def debug_hold_sms(n_ctas: int, ns: int, stream: torch.cuda.Stream) -> None:
    """Test only: occupy n_ctas SMs for ns nanoseconds on `stream` (readme_debug_hold_sms)."""
    lib().readme_set_device(stream.device.index)
    _check("readme_debug_hold_sms", lib().readme_debug_hold_sms(int(n_ctas), int(ns), ctypes.c_void_p(stream.cuda_stream)))
