"""Thin binding of the DCNv4 module path (include/dcnv4_module.h).

PAPER.md P:334: the offset and modulation linear layers are "combined into one linear
layer"; the lightweight module has no input/output projections, so the
operator samples the module input.  `offset_mask_linear` is that fused linear on the
sm_100a tensor cores (dcnv4_offset_mask_linear); `module_forward` chains it with
dcnv4_forward.  Argument marshalling only: every step runs in libdcnv4.so's kernels, and
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from .binding import DTYPE_CODE, _check, _check_buffer, _check_tensors, _ptr, _stream_ptr, lib, make_params
from .binding import forward as dcnv4_forward
from .binding import output_size

_bound = False


def _lib():
    global _bound
    L = lib()
    if not _bound:
        VP = ctypes.c_void_p
        from .binding import Params
        L.dcnv4_offset_mask_linear.argtypes = [ctypes.POINTER(Params), ctypes.c_int, ctypes.c_int32,
                                               VP, VP, VP, VP, VP]
        L.dcnv4_offset_mask_linear.restype = ctypes.c_int
        L.dcnv4_module_forward.argtypes = [ctypes.POINTER(Params), ctypes.c_int, VP, VP, VP, VP, VP]
        L.dcnv4_module_forward.restype = ctypes.c_int
        _bound = True
    return L


def _check_linear(weight: torch.Tensor, bias: Optional[torch.Tensor], group: int, C: int, K: int):
    """weight [3*G*K, C] (nn.Linear layout), bias [3*G*K] (R21)."""
    J = 3 * group * K
    if tuple(weight.shape) != (J, C):
        raise ValueError(f"weight is {tuple(weight.shape)}, expected [3*G*K, C] = [{J}, {C}]")
    if bias is not None and tuple(bias.shape) != (J,):
        raise ValueError(f"bias is {tuple(bias.shape)}, expected [{J}]")


def om_stride_for(G: int, K: int = 9, multiple: int = 8) -> int:
    """Padded offset_mask row length: 3*G*K rounded up to `multiple` channels (16-B rows)."""
    return -(-3 * G * K // multiple) * multiple


def offset_mask_linear(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor],
                       group: int, om_stride: Optional[int] = None, kernel_size=3,
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """offset_mask [N, H, W, S] = x [N, H, W, C] . weight[J, C]^T + bias (J = 3*G*K), columns
    J..S-1 zero; stride-1 'same' geometry (the linear reads x at every output pixel)."""
    ts = [x, weight] + ([bias] if bias is not None else [])
    _check_tensors(*ts)
    N, H, W, C = x.shape
    kh, kw = (kernel_size, kernel_size) if isinstance(kernel_size, int) else kernel_size
    S = om_stride if om_stride else om_stride_for(group, kh * kw)
    if C % group:
        raise ValueError(f"C = {C} is not divisible by group = {group}")
    _check_linear(weight, bias, group, C, kh * kw)
    p = make_params(N, H, W, group, C // group, (kh, kw), 1, ((kh - 1) // 2, (kw - 1) // 2), 1,
                    1.0, S)
    Ho, Wo = output_size(p)
    if (Ho, Wo) != (H, W):
        raise ValueError("offset_mask_linear needs a 'same' geometry (odd kernel)")
    if out is None:
        out = torch.empty((N, H, W, S), dtype=x.dtype, device=x.device)
    _check_buffer(out, (N, H, W, S), x, "out")
    with torch.cuda.device(x.device):
        _check(_lib().dcnv4_offset_mask_linear(ctypes.byref(p), DTYPE_CODE[x.dtype], C, _ptr(x),
                                               _ptr(weight), _ptr(bias), _ptr(out),
                                               ctypes.c_void_p(_stream_ptr(x))))
    return out


def module_forward(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor], group: int,
                   offset_scale=1.0, om_stride: Optional[int] = None,
                   om_out: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None):
    """Lightweight DCNv4 module forward (3x3, stride 1, pad 1): om = linear(x) on the
    tensor cores, then y = DCNv4(x, om).  Returns y."""
    om = offset_mask_linear(x, weight, bias, group, om_stride, out=om_out)
    return dcnv4_forward(x, om, group, 3, 1, 1, 1, offset_scale, out=out)


def forward_fused(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor], group: int,
                  offset_scale=1.0, softmax=False, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Fused lightweight DCNv4 module forward (3x3, stride 1, pad 1), ONE kernel
    (dcnv4_module_forward): each 16x8-pixel tile's offset_mask is computed on the tensor
    cores and consumed from shared memory, never written to memory."""
    ts = [x, weight] + ([bias] if bias is not None else [])
    _check_tensors(*ts)
    N, H, W, C = x.shape
    if C % group:
        raise ValueError(f"C = {C} is not divisible by group = {group}")
    _check_linear(weight, bias, group, C, 9)
    p = make_params(N, H, W, group, C // group, 3, 1, 1, 1, offset_scale, 0, softmax)
    if out is None:
        out = torch.empty_like(x)
    _check_buffer(out, x.shape, x, "out")
    with torch.cuda.device(x.device):
        _check(_lib().dcnv4_module_forward(ctypes.byref(p), DTYPE_CODE[x.dtype], _ptr(x), _ptr(weight),
                                           _ptr(bias), _ptr(out), ctypes.c_void_p(_stream_ptr(x))))
    return out
