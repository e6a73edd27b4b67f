"""Thin binding of the DCNv4 module path (include/dcnv4_module.h).

PAPER.md P:334: the offset and modulation linear layers are "combined into one linear
layer"; the lightweight module has no input/output projections, so the
operator samples the module input.  `offset_mask_linear` is that fused linear on the
sm_100a tensor cores (dcnv4_offset_mask_linear); `module_forward` chains it with
dcnv4_forward; `forward_fused` is the one-kernel lightweight module.  The full module
(1x1 input/output projections around the aggregation; R22)
is `full_forward` / `full_backward` / `DCNv4Module`, built from the tcgen05 GEMMs of
csrc/gemm.cu (`linear`, `linear_grad_input`, `linear_grad_weight`) and the fused
kernel with a separate value tensor (`core_forward`).  Argument marshalling only: every
step runs in libdcnv4.so's kernels, and there is no CPU fallback.
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


# ---------------------------------------------------------------------------------------
# The full DCNv4 module (R22) and its backward.
# Every step is one libdcnv4.so call (tcgen05 GEMMs in csrc/gemm.cu, the fused
# offset/mask + aggregation kernel, the DCNv4 backward); this file only marshals them.

_gbound = False


def _glib():
    global _gbound
    L = _lib()
    if not _gbound:
        VP, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        from .binding import Params
        L.dcnv4_module_core_forward.argtypes = [ctypes.POINTER(Params), ctypes.c_int, VP, VP, VP, VP, VP, VP]
        L.dcnv4_module_core_forward.restype = ctypes.c_int
        L.dcnv4_linear.argtypes = [ctypes.c_int, i64, i32, i32, VP, VP, VP, VP, VP]
        L.dcnv4_linear.restype = ctypes.c_int
        L.dcnv4_linear_grad_input.argtypes = [ctypes.c_int, i64, i32, i32, VP, i32, VP, i32, VP, VP, VP, VP]
        L.dcnv4_linear_grad_input.restype = ctypes.c_int
        L.dcnv4_linear_grad_weight_workspace_bytes.argtypes = [i32, i32]
        L.dcnv4_linear_grad_weight_workspace_bytes.restype = ctypes.c_size_t
        L.dcnv4_linear_grad_weight.argtypes = [ctypes.c_int, i64, i32, i32, VP, VP, i32, VP, VP, VP,
                                               ctypes.c_size_t, VP]
        L.dcnv4_linear_grad_weight.restype = ctypes.c_int
        _gbound = True
    return L


def _rows(t: torch.Tensor):
    return t.numel() // t.shape[-1]


def linear(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor] = None,
           out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """y[..., N] = x[..., K] . weight[N, K]^T + bias (dcnv4_linear, tcgen05)."""
    _check_tensors(*([x, weight] + ([bias] if bias is not None else [])))
    K, N = x.shape[-1], weight.shape[0]
    if tuple(weight.shape) != (N, K) or (bias is not None and tuple(bias.shape) != (N,)):
        raise ValueError(f"weight {tuple(weight.shape)} / bias must be [N, {K}] / [N]")
    shape = tuple(x.shape[:-1]) + (N,)
    if out is None:
        out = torch.empty(shape, dtype=x.dtype, device=x.device)
    _check_buffer(out, shape, x, "out")
    with torch.cuda.device(x.device):
        _check(_glib().dcnv4_linear(DTYPE_CODE[x.dtype], _rows(x), K, N, _ptr(x), _ptr(weight), _ptr(bias),
                                    _ptr(out), ctypes.c_void_p(_stream_ptr(x))))
    return out


def linear_grad_input(gy0: torch.Tensor, weight0: torch.Tensor, n0: Optional[int] = None,
                      gy1: Optional[torch.Tensor] = None, weight1: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """gx = gy0[..., :n0] . weight0 (+ gy1 . weight1) (dcnv4_linear_grad_input): the
    grad_input of one or two linear layers that read the same input."""
    ts = [gy0, weight0] + ([gy1, weight1] if gy1 is not None else [])
    _check_tensors(*ts)
    N0 = weight0.shape[0] if n0 is None else n0
    K = weight0.shape[1]
    N1 = weight1.shape[0] if gy1 is not None else 0
    if weight0.shape[0] != N0 or gy0.shape[-1] < N0:
        raise ValueError("gy0 / weight0 shapes disagree")
    if gy1 is not None and (tuple(weight1.shape) != (N1, K) or gy1.shape[-1] != N1
                            or _rows(gy1) != _rows(gy0)):
        raise ValueError("gy1 / weight1 shapes disagree")
    shape = tuple(gy0.shape[:-1]) + (K,)
    if out is None:
        out = torch.empty(shape, dtype=gy0.dtype, device=gy0.device)
    _check_buffer(out, shape, gy0, "out")
    with torch.cuda.device(gy0.device):
        _check(_glib().dcnv4_linear_grad_input(DTYPE_CODE[gy0.dtype], _rows(gy0), K, N0, _ptr(gy0), gy0.shape[-1],
                                               _ptr(weight0), N1, _ptr(gy1), _ptr(weight1), _ptr(out),
                                               ctypes.c_void_p(_stream_ptr(gy0))))
    return out


def linear_grad_weight(x: torch.Tensor, gy: torch.Tensor, n: Optional[int] = None, with_bias: bool = True,
                       workspace: Optional[torch.Tensor] = None):
    """(grad_weight [N, K], grad_bias [N] or None) of y = x . W^T + b over all rows
    (dcnv4_linear_grad_weight); gy may carry padding columns beyond n."""
    _check_tensors(x, gy)
    K = x.shape[-1]
    N = gy.shape[-1] if n is None else n
    if _rows(x) != _rows(gy) or gy.shape[-1] < N:
        raise ValueError("x / gy rows disagree")
    gw = torch.empty((N, K), dtype=x.dtype, device=x.device)
    gb = torch.empty((N,), dtype=x.dtype, device=x.device) if with_bias else None
    L = _glib()
    need = int(L.dcnv4_linear_grad_weight_workspace_bytes(K, N))
    from .binding import _workspace
    workspace = _workspace(workspace, need, x)
    with torch.cuda.device(x.device):
        _check(L.dcnv4_linear_grad_weight(DTYPE_CODE[x.dtype], _rows(x), K, N, _ptr(x), _ptr(gy), gy.shape[-1],
                                          _ptr(gw), _ptr(gb), _ptr(workspace), ctypes.c_size_t(need),
                                          ctypes.c_void_p(_stream_ptr(x))))
    return gw, gb


def core_forward(x: torch.Tensor, value: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor],
                 group: int, offset_scale=1.0, softmax=False, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """y = DCNv4(value, RN_T(x . weight^T + bias)) in ONE kernel (dcnv4_module_core_forward):
    the offset_mask from the module input x, the samples from `value` (R22)."""
    ts = [x, value, weight] + ([bias] if bias is not None else [])
    _check_tensors(*ts)
    N, H, W, C = x.shape
    if C % group:
        raise ValueError(f"C = {C} is not divisible by group = {group}")
    _check_buffer(value, x.shape, x, "value")
    _check_linear(weight, bias, group, C, 9)
    p = make_params(N, H, W, group, C // group, 3, 1, 1, 1, offset_scale, 0, softmax)
    if out is None:
        out = torch.empty_like(x)
    _check_buffer(out, x.shape, x, "out")
    with torch.cuda.device(x.device):
        _check(_glib().dcnv4_module_core_forward(ctypes.byref(p), DTYPE_CODE[x.dtype], _ptr(x), _ptr(value),
                                                 _ptr(weight), _ptr(bias), _ptr(out),
                                                 ctypes.c_void_p(_stream_ptr(x))))
    return out


FULL_KEYS = ("w_in", "b_in", "w_om", "b_om", "w_out", "b_out")


def full_forward(x: torch.Tensor, params: dict, group: int, offset_scale=1.0, softmax=False):
    """Full DCNv4 module forward (R22): v = linear(x; W_in), a = DCNv4(v, linear(x; W_om))
    fused in one kernel (f16/bf16; fp32: offset_mask linear + dcnv4_forward), y =
    linear(a; W_out).  Three launches (fp32: four).  Returns (y, (v, a)) --
    the saved activations of full_backward (the offset_mask is recomputed there)."""
    v = linear(x, params["w_in"], params.get("b_in"))
    if x.dtype == torch.float32:
        # fp32: 3xTF32 GEMMs (csrc/gemm.cu) and the fp32 operator; the offset_mask goes
        # through memory (the fused kernel's tensor-core linear is f16/bf16)
        om = linear(x, params["w_om"], params.get("b_om"))
        a = dcnv4_forward(v, om, group, 3, 1, 1, 1, offset_scale, softmax)
    else:
        a = core_forward(x, v, params["w_om"], params.get("b_om"), group, offset_scale, softmax)
    y = linear(a, params["w_out"], params.get("b_out"))
    return y, (v, a)


def full_backward(x: torch.Tensor, params: dict, group: int, gy: torch.Tensor, saved, offset_scale=1.0,
                  softmax=False) -> dict:
    """Backward of full_forward given gy: ga = gy . W_out; dW_out, db_out; the offset_mask
    recomputed (dcnv4_offset_mask_linear); (gv, gom) = dcnv4_backward(v, om, ga);
    gx = gv . W_in + gom . W_om (one GEMM over two K segments); dW_in, db_in, dW_om, db_om.
    Returns {"x": gx, "w_in": ..., "b_in": ..., ...}."""
    from .binding import backward as dcnv4_backward
    v, a = saved
    g = {}
    g["w_out"], g["b_out"] = linear_grad_weight(a, gy, with_bias=params.get("b_out") is not None)
    ga = linear_grad_input(gy, params["w_out"])
    if x.dtype == torch.float32:
        om = linear(x, params["w_om"], params.get("b_om"))  # [.., 3GK], S = 3GK
    else:
        om = offset_mask_linear(x, params["w_om"], params.get("b_om"), group, om_stride_for(group))
    gv, gom = dcnv4_backward(v, om, ga, group, 3, 1, 1, 1, offset_scale, softmax)
    J = params["w_om"].shape[0]
    g["x"] = linear_grad_input(gom, params["w_om"], J, gv, params["w_in"])
    g["w_in"], g["b_in"] = linear_grad_weight(x, gv, with_bias=params.get("b_in") is not None)
    g["w_om"], g["b_om"] = linear_grad_weight(x, gom, J, with_bias=params.get("b_om") is not None)
    return g


class FullModuleFunction(torch.autograd.Function):
    """Autograd wrapper of full_forward / full_backward."""

    @staticmethod
    def forward(ctx, x, w_in, b_in, w_om, b_om, w_out, b_out, group, offset_scale, softmax):
        params = dict(zip(FULL_KEYS, (w_in, b_in, w_om, b_om, w_out, b_out)))
        y, saved = full_forward(x, params, group, offset_scale, softmax)
        ctx.cfg = (group, offset_scale, softmax)
        ctx.has_bias = tuple(params[k] is not None for k in ("b_in", "b_om", "b_out"))
        ctx.save_for_backward(x, w_in, b_in, w_om, b_om, w_out, b_out, *saved)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, w_in, b_in, w_om, b_om, w_out, b_out, v, a = ctx.saved_tensors
        params = dict(zip(FULL_KEYS, (w_in, b_in, w_om, b_om, w_out, b_out)))
        group, offset_scale, softmax = ctx.cfg
        g = full_backward(x, params, group, gy.contiguous(), (v, a), offset_scale, softmax)
        return (g["x"], g["w_in"], g["b_in"], g["w_om"], g["b_om"], g["w_out"], g["b_out"], None, None, None)


class DCNv4Module(torch.nn.Module):
    """The full DCNv4 module on NHWC inputs [N, H, W, C]:
    3x3 kernel, stride 1, pad 1; G groups of D = C / G channels; F16/BF16 parameters."""

    def __init__(self, channels: int, group: int, offset_scale: float = 1.0, softmax: bool = False,
                 dtype=torch.float16, device="cuda"):
        super().__init__()
        C, J = channels, 27 * group
        kw = dict(dtype=dtype, device=device)
        self.group, self.offset_scale, self.softmax = group, offset_scale, softmax
        self.w_in = torch.nn.Parameter(torch.empty(C, C, **kw))
        self.b_in = torch.nn.Parameter(torch.zeros(C, **kw))
        self.w_om = torch.nn.Parameter(torch.zeros(J, C, **kw))  # DCNv3/v4 init: zero offsets
        self.b_om = torch.nn.Parameter(torch.zeros(J, **kw))
        self.w_out = torch.nn.Parameter(torch.empty(C, C, **kw))
        self.b_out = torch.nn.Parameter(torch.zeros(C, **kw))
        torch.nn.init.xavier_uniform_(self.w_in)
        torch.nn.init.xavier_uniform_(self.w_out)

    def forward(self, x):
        return FullModuleFunction.apply(x, self.w_in, self.b_in, self.w_om, self.b_om, self.w_out, self.b_out,
                                        self.group, self.offset_scale, self.softmax)
