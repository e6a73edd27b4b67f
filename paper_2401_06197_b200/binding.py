"""Thin Python binding of libdcnv4.so (include/dcnv4.h): argument marshalling only.

Every step of the operator runs in the library's CUDA kernels; PyTorch supplies device
memory, the current stream and autograd plumbing.  There is no CPU fallback: if the
shared library is missing or a call fails, an exception is raised.

Operator (Eq. (1)-(2), DCNv4 = no softmax):
    y[n, ho, wo, g*D + c] = sum_k m_k * bilinear(x[n, :, :, g*D + c], p0 + p_k + dp_k)
Layouts: x [N, H, W, G*D]; offset_mask [N, Ho, Wo, S] with per-group rows
[dx_0, dy_0, ..., dx_{K-1}, dy_{K-1}, m_0, ..., m_{K-1}] (include/dcnv4.h).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# DCNV4_LIB: path of an alternative build of the library (A/B experiments,
# scripts/build_variant.py); the in-tree libdcnv4.so otherwise
LIB_PATH = os.environ.get("DCNV4_LIB") or os.path.join(_HERE, "libdcnv4.so")

OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_UNSUPPORTED, ERR_MISALIGNED, ERR_WORKSPACE, ERR_CUDA = range(7)
_STATUS = {1: "INVALID_ARG", 2: "SHAPE", 3: "UNSUPPORTED", 4: "MISALIGNED", 5: "WORKSPACE",
           6: "CUDA"}
DTYPE_CODE = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}


class DCNv4Error(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"DCNV4_ERR_{_STATUS.get(status, status)}: {message}")
        self.status = status


class Params(ctypes.Structure):
    """Mirror of dcnv4_params."""
    _fields_ = [("N", ctypes.c_int64), ("H", ctypes.c_int64), ("W", ctypes.c_int64),
                ("G", ctypes.c_int32), ("D", ctypes.c_int32),
                ("kernel_h", ctypes.c_int32), ("kernel_w", ctypes.c_int32),
                ("stride_h", ctypes.c_int32), ("stride_w", ctypes.c_int32),
                ("pad_h", ctypes.c_int32), ("pad_w", ctypes.c_int32),
                ("dilation_h", ctypes.c_int32), ("dilation_w", ctypes.c_int32),
                ("offset_scale", ctypes.c_float), ("om_stride", ctypes.c_int32),
                ("softmax", ctypes.c_int32), ("deterministic", ctypes.c_int32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdcnv4.so (built by __graft_entry__.build() / _build.py); fail loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P, VP = ctypes.POINTER(Params), ctypes.c_void_p
        L.dcnv4_version.restype = ctypes.c_int
        L.dcnv4_last_error.restype = ctypes.c_char_p
        L.dcnv4_output_size.argtypes = [P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.dcnv4_forward.argtypes = [P, ctypes.c_int, VP, VP, VP, VP]
        L.dcnv4_backward_workspace_bytes.argtypes = [P, ctypes.c_int]
        L.dcnv4_backward_workspace_bytes.restype = ctypes.c_size_t
        L.dcnv4_backward.argtypes = [P, ctypes.c_int, VP, VP, VP, VP, VP, VP, ctypes.c_size_t, VP]
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.dcnv4_launch_info.argtypes = [P, ctypes.c_int, ctypes.c_int, i32p, i32p, i32p, i32p,
                                        ctypes.POINTER(ctypes.c_int64)]
        PP = ctypes.POINTER(ctypes.POINTER(Params))
        VPP = ctypes.POINTER(ctypes.c_void_p)
        L.dcnv4_forward_grouped.argtypes = [PP, ctypes.c_int32, ctypes.c_int, VPP, VPP, VPP, VP]
        for fn in ("dcnv4_output_size", "dcnv4_forward", "dcnv4_backward", "dcnv4_launch_info",
                   "dcnv4_forward_grouped"):
            getattr(L, fn).restype = ctypes.c_int
        _lib = L
    return _lib


def _pair(v):
    return (int(v), int(v)) if isinstance(v, int) else (int(v[0]), int(v[1]))


def make_params(N, H, W, G, D, kernel_size=3, stride=1, pad=1, dilation=1, offset_scale=1.0,
                om_stride=0, softmax=False, deterministic=False) -> Params:
    kh, kw = _pair(kernel_size)
    sh, sw = _pair(stride)
    ph, pw = _pair(pad)
    dh, dw = _pair(dilation)
    return Params(N, H, W, G, D, kh, kw, sh, sw, ph, pw, dh, dw, float(offset_scale),
                  int(om_stride), int(bool(softmax)), int(bool(deterministic)))


def _check(rc: int):
    if rc != OK:
        raise DCNv4Error(rc, lib().dcnv4_last_error().decode())


def output_size(p: Params) -> Tuple[int, int]:
    ho, wo = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().dcnv4_output_size(ctypes.byref(p), ctypes.byref(ho), ctypes.byref(wo)))
    return ho.value, wo.value


def om_channels(p: Params) -> int:
    return p.om_stride if p.om_stride else 3 * p.G * p.kernel_h * p.kernel_w


def launch_info(p: Params, dtype: torch.dtype, backward: bool = False) -> dict:
    a, b, c, d = (ctypes.c_int32() for _ in range(4))
    e = ctypes.c_int64()
    _check(lib().dcnv4_launch_info(ctypes.byref(p), DTYPE_CODE[dtype], int(backward),
                                   ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                   ctypes.byref(d), ctypes.byref(e)))
    return {"lanes": a.value, "chunks_per_lane": b.value, "pixels_per_cta": c.value,
            "threads_per_cta": d.value, "ctas": e.value}


def _stream_ptr(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _params_for(x: torch.Tensor, om: torch.Tensor, G: int, kernel_size, stride, pad, dilation,
                offset_scale, softmax, deterministic=False) -> Params:
    if x.dim() != 4 or om.dim() != 4:
        raise ValueError("x must be [N,H,W,C] and offset_mask [N,Ho,Wo,S]")
    N, H, W, C = x.shape
    if C % G:
        raise ValueError(f"C = {C} is not divisible by group = {G}")
    p = make_params(N, H, W, G, C // G, kernel_size, stride, pad, dilation, offset_scale,
                    om.shape[3], softmax, deterministic)
    Ho, Wo = output_size(p)
    if tuple(om.shape[:3]) != (N, Ho, Wo):
        raise ValueError(f"offset_mask is {tuple(om.shape)}, expected [{N}, {Ho}, {Wo}, S]")
    return p


def _check_tensors(*ts):
    dev = ts[0].device
    for t in ts:
        if not t.is_cuda:
            raise ValueError("dcnv4 tensors must be CUDA tensors (no CPU fallback)")
        if t.device != dev:
            raise ValueError("all tensors must be on the same device")
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
        if t.dtype != ts[0].dtype:
            raise ValueError("all tensors must share one dtype")
    if ts[0].dtype not in DTYPE_CODE:
        raise ValueError(f"unsupported dtype {ts[0].dtype}")


def _check_buffer(t: torch.Tensor, shape, like: torch.Tensor, name: str):
    """A caller-supplied output buffer: exact shape, the inputs' dtype and device,
    contiguous (the kernels and TMA maps size everything from the params)."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} is {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != like.dtype:
        raise ValueError(f"{name} has dtype {t.dtype}, expected {like.dtype}")
    if t.device != like.device:
        raise ValueError(f"{name} is on {t.device}, expected {like.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _workspace(workspace: Optional[torch.Tensor], need: int, like: torch.Tensor):
    """A caller-supplied scratch buffer (any dtype, >= need bytes, same device,
    contiguous), or a fresh one."""
    if not need:
        return None
    if workspace is None:
        return torch.empty(need, dtype=torch.uint8, device=like.device)
    if workspace.device != like.device:
        raise ValueError(f"workspace is on {workspace.device}, expected {like.device}")
    if not workspace.is_contiguous():
        raise ValueError("workspace must be contiguous")
    if workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"workspace has {workspace.numel() * workspace.element_size()} bytes, "
                         f"{need} required")
    return workspace


def forward(x: torch.Tensor, offset_mask: torch.Tensor, group: int, kernel_size=3, stride=1,
            pad=1, dilation=1, offset_scale=1.0, softmax=False,
            out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """y = DCNv4(x, offset_mask): one dcnv4_forward call on the current stream."""
    _check_tensors(x, offset_mask)
    p = _params_for(x, offset_mask, group, kernel_size, stride, pad, dilation, offset_scale,
                    softmax)
    Ho, Wo = output_size(p)
    if out is None:
        out = torch.empty((x.shape[0], Ho, Wo, x.shape[3]), dtype=x.dtype, device=x.device)
    _check_buffer(out, (x.shape[0], Ho, Wo, x.shape[3]), x, "out")
    with torch.cuda.device(x.device):
        _check(lib().dcnv4_forward(ctypes.byref(p), DTYPE_CODE[x.dtype], _ptr(x),
                                   _ptr(offset_mask), _ptr(out), ctypes.c_void_p(_stream_ptr(x))))
    return out


def forward_grouped(xs, offset_masks, groups, kernel_size=3, stride=1, pad=1, dilation=1,
                    offset_scale=1.0, softmax=False, outs=None):
    """[DCNv4(x_i, om_i)] for up to 8 independent problems in one dcnv4_forward_grouped call
    (one persistent launch when they share the kernel instantiation and tile shape)."""
    n = len(xs)
    if not (len(offset_masks) == n and len(groups) == n and 1 <= n <= 8):
        raise ValueError("xs, offset_masks, groups must have the same length in [1, 8]")
    _check_tensors(*xs, *offset_masks)
    ps = [_params_for(x, om, G, kernel_size, stride, pad, dilation, offset_scale, softmax)
          for x, om, G in zip(xs, offset_masks, groups)]
    if outs is None:
        outs = []
        for x, p in zip(xs, ps):
            Ho, Wo = output_size(p)
            outs.append(torch.empty((x.shape[0], Ho, Wo, x.shape[3]), dtype=x.dtype, device=x.device))
    for x, p, o in zip(xs, ps, outs):
        Ho, Wo = output_size(p)
        _check_buffer(o, (x.shape[0], Ho, Wo, x.shape[3]), x, "out")
    parr = (ctypes.POINTER(Params) * n)(*[ctypes.pointer(p) for p in ps])
    vp = lambda ts: (ctypes.c_void_p * n)(*[t.data_ptr() for t in ts])  # noqa: E731
    with torch.cuda.device(xs[0].device):
        _check(lib().dcnv4_forward_grouped(parr, n, DTYPE_CODE[xs[0].dtype], vp(xs), vp(offset_masks), vp(outs),
                                           ctypes.c_void_p(_stream_ptr(xs[0]))))
    return outs


def workspace_bytes(p: Params, dtype: torch.dtype) -> int:
    return int(lib().dcnv4_backward_workspace_bytes(ctypes.byref(p), DTYPE_CODE[dtype]))


def backward(x: torch.Tensor, offset_mask: torch.Tensor, grad_output: torch.Tensor, group: int,
             kernel_size=3, stride=1, pad=1, dilation=1, offset_scale=1.0, softmax=False,
             grad_input: Optional[torch.Tensor] = None,
             grad_offset_mask: Optional[torch.Tensor] = None,
             workspace: Optional[torch.Tensor] = None, deterministic=False):
    """(grad_input, grad_offset_mask): one dcnv4_backward call on the current stream.
    deterministic=True: bit-reproducible grad_input (int64 fixed point, R19)."""
    _check_tensors(x, offset_mask, grad_output)
    p = _params_for(x, offset_mask, group, kernel_size, stride, pad, dilation, offset_scale,
                    softmax, deterministic)
    Ho, Wo = output_size(p)
    _check_buffer(grad_output, (x.shape[0], Ho, Wo, x.shape[3]), x, "grad_output")
    if grad_input is None:
        grad_input = torch.empty_like(x)
    if grad_offset_mask is None:
        grad_offset_mask = torch.empty_like(offset_mask)
    _check_buffer(grad_input, x.shape, x, "grad_input")
    _check_buffer(grad_offset_mask, offset_mask.shape, x, "grad_offset_mask")
    need = workspace_bytes(p, x.dtype)
    workspace = _workspace(workspace, need, x)
    with torch.cuda.device(x.device):
        _check(lib().dcnv4_backward(ctypes.byref(p), DTYPE_CODE[x.dtype], _ptr(x),
                                    _ptr(offset_mask), _ptr(grad_output), _ptr(grad_input),
                                    _ptr(grad_offset_mask), _ptr(workspace) if need else None,
                                    ctypes.c_size_t(need), ctypes.c_void_p(_stream_ptr(x))))
    return grad_input, grad_offset_mask


class DCNv4Function(torch.autograd.Function):
    """Autograd wrapper: forward = dcnv4_forward, backward = dcnv4_backward."""

    @staticmethod
    def forward(ctx, x, offset_mask, group, kernel_size, stride, pad, dilation, offset_scale,
                softmax, deterministic=False):
        ctx.cfg = (group, kernel_size, stride, pad, dilation, offset_scale, softmax)
        ctx.deterministic = bool(deterministic)
        ctx.save_for_backward(x, offset_mask)
        return forward(x, offset_mask, group, kernel_size, stride, pad, dilation, offset_scale,
                       softmax)

    @staticmethod
    def backward(ctx, gy):
        x, om = ctx.saved_tensors
        gx, gom = backward(x, om, gy.contiguous(), *ctx.cfg, deterministic=ctx.deterministic)
        return gx, gom, None, None, None, None, None, None, None, None


def dcnv4(x, offset_mask, group, kernel_size=3, stride=1, pad=1, dilation=1, offset_scale=1.0,
          softmax=False, deterministic=False):
    """Differentiable DCNv4 spatial aggregation (the paper's core operator).
    deterministic=True makes the backward's grad_input bit-reproducible."""
    return DCNv4Function.apply(x, offset_mask, group, kernel_size, stride, pad, dilation,
                               offset_scale, softmax, deterministic)
