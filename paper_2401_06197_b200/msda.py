"""Thin Python binding of the multi-scale deformable attention entry points of
libdcnv4.so (include/msda.h): argument marshalling only, no CPU
fallback.

    out[n, q, m, :] = sum_{l, p} attn[n, q, m, l, p] * V_l[n, :, m, :](phi_l(loc[n, q, m, l, p]))
    value [N, S, M, D] (levels flattened, S = sum H_l*W_l), loc [N, Lq, M, L, P, 2] (x, y)
    normalised to [0, 1], attn [N, Lq, M, L, P], out [N, Lq, M, D].
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import torch

from .binding import DTYPE_CODE, _check, _check_buffer, _check_tensors, _ptr, _stream_ptr, _workspace, lib

MAX_LEVELS = 8


class MSDAParams(ctypes.Structure):
    """Mirror of msda_params."""
    _fields_ = [("N", ctypes.c_int64), ("Lq", ctypes.c_int64),
                ("M", ctypes.c_int32), ("D", ctypes.c_int32),
                ("L", ctypes.c_int32), ("P", ctypes.c_int32),
                ("H", ctypes.c_int32 * MAX_LEVELS), ("W", ctypes.c_int32 * MAX_LEVELS)]


_ready = False


def _lib():
    global _ready
    L = lib()
    if not _ready:
        P, VP = ctypes.POINTER(MSDAParams), ctypes.c_void_p
        L.msda_value_tokens.argtypes = [P, ctypes.POINTER(ctypes.c_int64)]
        L.msda_forward.argtypes = [P, ctypes.c_int, VP, VP, VP, VP, VP]
        L.msda_backward_workspace_bytes.argtypes = [P, ctypes.c_int]
        L.msda_backward_workspace_bytes.restype = ctypes.c_size_t
        L.msda_backward.argtypes = [P, ctypes.c_int, VP, VP, VP, VP, VP, VP, VP, VP,
                                    ctypes.c_size_t, VP]
        for fn in ("msda_value_tokens", "msda_forward", "msda_backward"):
            getattr(L, fn).restype = ctypes.c_int
        _ready = True
    return L


def make_params(N: int, Lq: int, M: int, D: int, P: int,
                shapes: Sequence[Tuple[int, int]]) -> MSDAParams:
    if len(shapes) > MAX_LEVELS:
        raise ValueError(f"at most {MAX_LEVELS} levels")
    H = (ctypes.c_int32 * MAX_LEVELS)(*([h for h, _ in shapes] + [0] * (MAX_LEVELS - len(shapes))))
    W = (ctypes.c_int32 * MAX_LEVELS)(*([w for _, w in shapes] + [0] * (MAX_LEVELS - len(shapes))))
    return MSDAParams(N, Lq, M, D, len(shapes), P, H, W)


def value_tokens(p: MSDAParams) -> int:
    s = ctypes.c_int64()
    _check(_lib().msda_value_tokens(ctypes.byref(p), ctypes.byref(s)))
    return s.value


def _params_for(value, loc, attn, shapes) -> MSDAParams:
    if value.dim() != 4 or loc.dim() != 6 or attn.dim() != 5:
        raise ValueError("value [N,S,M,D], loc [N,Lq,M,L,P,2], attn [N,Lq,M,L,P] expected")
    N, S, M, D = value.shape
    _, Lq, _, L, P, two = loc.shape
    if two != 2 or L != len(shapes) or tuple(attn.shape) != (N, Lq, M, L, P) or loc.shape[0] != N \
            or loc.shape[2] != M:
        raise ValueError(f"inconsistent shapes value {tuple(value.shape)} loc {tuple(loc.shape)} "
                         f"attn {tuple(attn.shape)} levels {len(shapes)}")
    p = make_params(N, Lq, M, D, P, shapes)
    if value_tokens(p) != S:
        raise ValueError(f"value has {S} tokens, the level shapes give {value_tokens(p)}")
    return p


def workspace_bytes(p: MSDAParams, dtype: torch.dtype) -> int:
    return int(_lib().msda_backward_workspace_bytes(ctypes.byref(p), DTYPE_CODE[dtype]))


def forward(value, loc, attn, shapes, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """out = MSDA(value, loc, attn): one msda_forward call on the current stream."""
    _check_tensors(value, loc, attn)
    p = _params_for(value, loc, attn, shapes)
    if out is None:
        out = torch.empty((p.N, p.Lq, p.M, p.D), dtype=value.dtype, device=value.device)
    _check_buffer(out, (p.N, p.Lq, p.M, p.D), value, "out")
    with torch.cuda.device(value.device):
        _check(_lib().msda_forward(ctypes.byref(p), DTYPE_CODE[value.dtype], _ptr(value), _ptr(loc),
                                   _ptr(attn), _ptr(out), ctypes.c_void_p(_stream_ptr(value))))
    return out


def backward(value, loc, attn, grad_out, shapes, grad_value=None, grad_loc=None,
             grad_attn=None, workspace=None):
    """(grad_value, grad_loc, grad_attn): one msda_backward call on the current stream."""
    _check_tensors(value, loc, attn, grad_out)
    p = _params_for(value, loc, attn, shapes)
    grad_value = torch.empty_like(value) if grad_value is None else grad_value
    grad_loc = torch.empty_like(loc) if grad_loc is None else grad_loc
    grad_attn = torch.empty_like(attn) if grad_attn is None else grad_attn
    _check_buffer(grad_out, (p.N, p.Lq, p.M, p.D), value, "grad_out")
    _check_buffer(grad_value, value.shape, value, "grad_value")
    _check_buffer(grad_loc, loc.shape, value, "grad_loc")
    _check_buffer(grad_attn, attn.shape, value, "grad_attn")
    need = workspace_bytes(p, value.dtype)
    workspace = _workspace(workspace, need, value)
    with torch.cuda.device(value.device):
        _check(_lib().msda_backward(ctypes.byref(p), DTYPE_CODE[value.dtype], _ptr(value), _ptr(loc),
                                    _ptr(attn), _ptr(grad_out), _ptr(grad_value), _ptr(grad_loc),
                                    _ptr(grad_attn), _ptr(workspace) if need else None,
                                    ctypes.c_size_t(need), ctypes.c_void_p(_stream_ptr(value))))
    return grad_value, grad_loc, grad_attn


class MSDAFunction(torch.autograd.Function):
    """Autograd wrapper: forward = msda_forward, backward = msda_backward."""

    @staticmethod
    def forward(ctx, value, loc, attn, shapes):
        ctx.shapes = tuple(tuple(s) for s in shapes)
        ctx.save_for_backward(value, loc, attn)
        return forward(value, loc, attn, ctx.shapes)

    @staticmethod
    def backward(ctx, gout):
        value, loc, attn = ctx.saved_tensors
        gv, gl, ga = backward(value, loc, attn, gout.contiguous(), ctx.shapes)
        return gv, gl, ga, None


def msda(value, loc, attn, shapes):
    """Differentiable multi-scale deformable attention sampling core."""
    return MSDAFunction.apply(value, loc, attn, shapes)
