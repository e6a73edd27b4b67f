"""The C-ABI library loads and exports every symbol include/dcnv4.h declares; host-only
entry points (no CUDA call) behave as documented.  CPU only."""
import ctypes
import os
import re

import pytest
import torch

import oracle
import paper_2401_06197_b200 as pkg
from paper_2401_06197_b200 import binding as b

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dcnv4.h")


MSDA_HEADER = os.path.join(ROOT, "include", "msda.h")
MODULE_HEADER = os.path.join(ROOT, "include", "dcnv4_module.h")


def _declared():
    out = []
    for h in (HEADER, MSDA_HEADER, MODULE_HEADER):
        src = open(h).read()
        out += re.findall(r"DCNV4_API\s+[\w\s\*]+?\b((?:dcnv4|msda)_\w+)\s*\(", src)
    return out


def test_header_declares_the_boundary():
    names = set(_declared())
    assert {"dcnv4_forward", "dcnv4_backward", "dcnv4_output_size", "dcnv4_last_error",
            "dcnv4_version", "dcnv4_backward_workspace_bytes", "dcnv4_launch_info"} <= names
    assert {"msda_forward", "msda_backward", "msda_value_tokens",
            "msda_backward_workspace_bytes"} <= names
    assert "dcnv4_offset_mask_linear" in names


def test_offset_mask_linear_validation():
    """Host-side checks of dcnv4_offset_mask_linear return before any CUDA call."""
    from paper_2401_06197_b200 import module
    lib = module._lib()
    p = b.make_params(1, 8, 8, 4, 16, 3, 1, 1, 1, 1.0, 112)
    args = (64, None, None, None, None, None)
    assert lib.dcnv4_offset_mask_linear(ctypes.byref(p), 0, *args) == b.ERR_UNSUPPORTED
    assert b"F32" in lib.dcnv4_last_error()
    assert lib.dcnv4_offset_mask_linear(ctypes.byref(p), 1, 60, *args[1:]) == b.ERR_UNSUPPORTED
    assert b"C_in" in lib.dcnv4_last_error()
    p2 = b.make_params(1, 8, 8, 4, 16, 3, 1, 1, 1, 1.0, 108)  # 108 % 8 != 0
    assert lib.dcnv4_offset_mask_linear(ctypes.byref(p2), 1, *args) == b.ERR_UNSUPPORTED
    assert b"om_stride" in lib.dcnv4_last_error()
    p3 = b.make_params(1, 8, 8, 4, 16, 3, 1, 1, 1, 1.0, 104)  # < 3GK
    assert lib.dcnv4_offset_mask_linear(ctypes.byref(p3), 1, *args) == b.ERR_SHAPE
    assert lib.dcnv4_offset_mask_linear(ctypes.byref(p), 1, *args) == b.ERR_INVALID_ARG
    assert b"feat" in lib.dcnv4_last_error()
    p0 = b.make_params(0, 8, 8, 4, 16, 3, 1, 1, 1, 1.0, 112)  # empty batch: no-op
    assert lib.dcnv4_offset_mask_linear(ctypes.byref(p0), 2, *args) == b.OK
    assert module.om_stride_for(4) == 112 and module.om_stride_for(32) == 864


def test_module_forward_validation():
    """Host-side checks of dcnv4_module_forward (no CUDA call before they pass)."""
    from paper_2401_06197_b200 import module
    lib = module._lib()
    ok = b.make_params(1, 8, 8, 4, 16, 3, 1, 1, 1)
    nul = (None, None, None, None, None)
    assert lib.dcnv4_module_forward(ctypes.byref(ok), 0, *nul) == b.ERR_UNSUPPORTED  # F32
    for bad in (b.make_params(1, 8, 8, 4, 16, 3, 2, 1, 1),   # stride 2
                b.make_params(1, 8, 8, 4, 16, 5, 1, 2, 1),   # 5x5
                b.make_params(1, 8, 8, 4, 16, 3, 1, 0, 1),   # pad 0
                b.make_params(1, 8, 8, 4, 16, 3, 1, 2, 2)):  # dilation 2
        assert lib.dcnv4_module_forward(ctypes.byref(bad), 1, *nul) == b.ERR_UNSUPPORTED
        assert b"3x3" in lib.dcnv4_last_error()
    d8 = b.make_params(1, 8, 8, 8, 8, 3, 1, 1, 1)  # D*2 = 16 B
    assert lib.dcnv4_module_forward(ctypes.byref(d8), 1, *nul) == b.ERR_UNSUPPORTED
    g3 = b.make_params(1, 8, 8, 3, 16, 3, 1, 1, 1)  # G not a multiple of GC = 4
    assert lib.dcnv4_module_forward(ctypes.byref(g3), 2, *nul) == b.ERR_UNSUPPORTED
    assert lib.dcnv4_module_forward(ctypes.byref(ok), 1, *nul) == b.ERR_INVALID_ARG
    assert b"input" in lib.dcnv4_last_error()
    mis = (ctypes.c_void_p(0x1008), ctypes.c_void_p(0x2000), None, ctypes.c_void_p(0x3000), None)
    assert lib.dcnv4_module_forward(ctypes.byref(ok), 1, *mis) == b.ERR_MISALIGNED
    empty = b.make_params(0, 8, 8, 4, 16, 3, 1, 1, 1)
    assert lib.dcnv4_module_forward(ctypes.byref(empty), 1, *nul) == b.OK


def test_msda_params_and_validation():
    from paper_2401_06197_b200 import msda
    assert ctypes.sizeof(msda.MSDAParams) == 96
    p = msda.make_params(2, 100, 8, 32, 4, [(10, 12), (5, 6), (3, 3), (2, 2)])
    assert msda.value_tokens(p) == 120 + 30 + 9 + 4
    assert msda.workspace_bytes(p, torch.float32) == 0
    assert msda.workspace_bytes(p, torch.bfloat16) == 2 * 163 * 8 * 32 * 4
    lib = pkg.lib()
    bad = msda.make_params(1, 4, 2, 6, 1, [(3, 3)])  # D*4 = 24 B
    assert lib.msda_forward(ctypes.byref(bad), 0, None, None, None, None, None) == b.ERR_UNSUPPORTED
    assert b"16" in lib.dcnv4_last_error()
    bad = msda.make_params(1, 4, 2, 8, 1, [(3, 0)])
    assert lib.msda_forward(ctypes.byref(bad), 0, None, None, None, None, None) == b.ERR_INVALID_ARG
    assert b"level 0" in lib.dcnv4_last_error()
    bad = msda.make_params(1, 4, 2, 8, 0, [(3, 3)])
    assert lib.msda_forward(ctypes.byref(bad), 0, None, None, None, None, None) == b.ERR_INVALID_ARG
    assert b"P" in lib.dcnv4_last_error()
    ok = msda.make_params(0, 4, 2, 8, 1, [(3, 3)])  # empty batch: no-op, no CUDA call
    assert lib.msda_forward(ctypes.byref(ok), 0, None, None, None, None, None) == b.OK


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(b.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert pkg.lib().dcnv4_version() == 130


def test_params_struct_layout():
    assert ctypes.sizeof(b.Params) == 80
    assert b.Params.offset_scale.offset == 64 and b.Params.softmax.offset == 72


@pytest.mark.parametrize("k,s,p,d", [((3, 3), (1, 1), (1, 1), (1, 1)), ((3, 3), (2, 2), (1, 1), (1, 1)),
                                     ((5, 3), (1, 2), (2, 0), (1, 2)), ((1, 1), (1, 1), (0, 0), (1, 1)),
                                     ((2, 2), (1, 1), (0, 1), (1, 1)), ((3, 3), (2, 1), (0, 2), (2, 2))])
def test_output_size_matches_conv_arithmetic(k, s, p, d):
    for H, W in [(7, 9), (56, 56), (200, 320), (1, 5)]:
        g = oracle.Geometry(N=2, H=H, W=W, G=2, D=16, kh=k[0], kw=k[1], sh=s[0], sw=s[1],
                            ph=p[0], pw=p[1], dh=d[0], dw=d[1])
        Ho, Wo = g.out_hw()
        prm = b.make_params(2, H, W, 2, 16, k, s, p, d)
        if Ho <= 0 or Wo <= 0:
            with pytest.raises(b.DCNv4Error):
                b.output_size(prm)
            continue
        assert b.output_size(prm) == (Ho, Wo)


def _status(fn, *args):
    return fn(*args)


def test_validation_errors_name_the_axis():
    L = pkg.lib()
    P = b.make_params
    cases = [
        (P(1, 8, 8, 2, 6), 0, b.ERR_UNSUPPORTED, "group channel"),    # 24 B not a multiple of 16
        (P(1, 8, 8, 2, 8), 1, b.OK, ""),                                 # f16 D=8 -> 16 B ok
        (P(1, 8, 8, 0, 16), 0, b.ERR_INVALID_ARG, "G"),
        (P(1, 0, 8, 2, 16), 0, b.ERR_INVALID_ARG, "H"),
        (P(1, 8, 8, 2, 16, om_stride=10), 0, b.ERR_SHAPE, "om_stride"),
        (P(1, 2, 2, 2, 16, kernel_size=5, pad=0), 0, b.ERR_SHAPE, "H axis"),
        (P(1, 8, 8, 2, 16, kernel_size=9), 0, b.ERR_UNSUPPORTED, "K"),
        (P(1, 8, 8, 2, 128), 0, b.ERR_UNSUPPORTED, "exceeds 256"),
        (P(1, 8, 8, 2, 16, offset_scale=float("nan")), 0, b.ERR_INVALID_ARG, "offset_scale"),
    ]
    for prm, dt, code, word in cases:
        rc = L.dcnv4_launch_info(ctypes.byref(prm), dt, 0, None, None, None, None, None)
        assert rc == code, (prm.D, prm.G, code, rc, L.dcnv4_last_error())
        if code:
            assert word in L.dcnv4_last_error().decode()
    assert L.dcnv4_forward(None, 0, None, None, None, None) == b.ERR_INVALID_ARG
    assert L.dcnv4_forward(ctypes.byref(P(1, 8, 8, 2, 16)), 7, None, None, None, None) == b.ERR_INVALID_ARG
    # NULL / misaligned pointers are rejected before any CUDA call
    prm = P(1, 8, 8, 2, 16)
    assert L.dcnv4_forward(ctypes.byref(prm), 0, None, ctypes.c_void_p(16), ctypes.c_void_p(16), None) == b.ERR_INVALID_ARG
    assert L.dcnv4_forward(ctypes.byref(prm), 0, ctypes.c_void_p(8), ctypes.c_void_p(16),
                           ctypes.c_void_p(16), None) == b.ERR_MISALIGNED
    # N = 0 is a no-op (no launch)
    assert L.dcnv4_forward(ctypes.byref(P(0, 8, 8, 2, 16)), 0, None, None, None, None) == b.OK
    assert L.dcnv4_backward(ctypes.byref(P(0, 8, 8, 2, 16)), 0, None, None, None, None, None,
                            None, 0, None) == b.OK


def test_workspace_contract():
    prm = b.make_params(2, 8, 8, 2, 16)
    import torch
    assert b.workspace_bytes(prm, torch.float32) == 0
    assert b.workspace_bytes(prm, torch.float16) == 2 * 8 * 8 * 32 * 4
    L = pkg.lib()
    rc = L.dcnv4_backward(ctypes.byref(b.make_params(1, 8, 8, 2, 16)), 1, ctypes.c_void_p(16),
                          ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16),
                          ctypes.c_void_p(16), None, 0, None)
    assert rc == b.ERR_WORKSPACE


def test_launch_shape():
    import torch
    # InternImage-T stage 1 (c2): C=64, G=4, D=16
    prm = b.make_params(64, 56, 56, 4, 16)
    fi = b.launch_info(prm, torch.float32)
    assert fi["lanes"] * fi["chunks_per_lane"] == 4   # 64 B per (pixel, group) = 4 chunks
    assert fi["threads_per_cta"] % 32 == 0 and fi["threads_per_cta"] <= 512
    assert fi["ctas"] * fi["pixels_per_cta"] >= 64 * 56 * 56
    hi = b.launch_info(prm, torch.float16)
    assert hi["lanes"] * hi["chunks_per_lane"] == 2
    # G = 80 (c5 stage 3) stays within one CTA per pixel
    big = b.launch_info(b.make_params(32, 16, 16, 80, 16), torch.bfloat16, backward=True)
    assert big["threads_per_cta"] <= 512


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The product package never imports the oracle, and refuses CPU tensors."""
    import torch
    pkg_dir = os.path.join(ROOT, "paper_2401_06197_b200")
    for dirpath, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("no oracle", ""), f
    with pytest.raises(ValueError):
        pkg.forward(torch.zeros(1, 4, 4, 32), torch.zeros(1, 4, 4, 54), group=2)


def test_gemm_and_grouped_validation_before_any_launch():
    """Host-side validation of the round-2 entry points (no CUDA call is reached)."""
    from paper_2401_06197_b200 import module as mod
    L = mod._glib()
    V = ctypes.c_void_p
    # dcnv4_linear: bad sizes, unsupported pitches, NULL and misaligned operands, M = 0
    assert L.dcnv4_linear(1, 10, 0, 8, V(16), V(16), None, V(16), None) == b.ERR_INVALID_ARG
    assert L.dcnv4_linear(1, 10, 12, 8, V(16), V(16), None, V(16), None) == b.ERR_UNSUPPORTED
    assert b"multiples of 8" in L.dcnv4_last_error()
    assert L.dcnv4_linear(0, 10, 6, 8, V(16), V(16), None, V(16), None) == b.ERR_UNSUPPORTED
    assert L.dcnv4_linear(1, 10, 16, 8, None, V(16), None, V(16), None) == b.ERR_INVALID_ARG
    assert b"x" in L.dcnv4_last_error()
    assert L.dcnv4_linear(1, 10, 16, 8, V(8), V(16), None, V(16), None) == b.ERR_MISALIGNED
    assert L.dcnv4_linear(1, 0, 16, 8, None, None, None, None, None) == b.OK
    assert L.dcnv4_linear(5, 10, 16, 8, V(16), V(16), None, V(16), None) == b.ERR_INVALID_ARG
    # grad_input: ld0 < N0, second segment without operands
    assert L.dcnv4_linear_grad_input(1, 10, 16, 24, V(16), 16, V(16), 0, None, None, V(16), None) == b.ERR_INVALID_ARG
    assert L.dcnv4_linear_grad_input(1, 10, 16, 8, V(16), 16, V(16), 8, None, None, V(16), None) == b.ERR_INVALID_ARG
    # grad_weight: the fp32 accumulator workspace is required and sized (N*K + N) * 4
    assert L.dcnv4_linear_grad_weight_workspace_bytes(64, 108) == (108 * 64 + 108) * 4
    assert L.dcnv4_linear_grad_weight(1, 10, 64, 108, V(16), V(16), 112, V(16), None, None, 0,
                                      None) == b.ERR_WORKSPACE
    assert L.dcnv4_linear_grad_weight(1, 10, 64, 108, V(16), V(16), 100, V(16), None, V(16), 10 ** 6,
                                      None) == b.ERR_INVALID_ARG  # ld_gy < N
    assert L.dcnv4_linear_grad_weight(1, 10, 64, 108, V(16), V(16), 116, V(16), None, V(16), 10 ** 6,
                                      None) == b.ERR_UNSUPPORTED  # ld_gy not 16-B
    # grouped forward: count bounds, NULL arrays, a bad problem named by index
    prm = b.make_params(1, 8, 8, 2, 16)
    PP = ctypes.POINTER(b.Params)
    arr = (PP * 2)(ctypes.pointer(prm), ctypes.pointer(b.make_params(1, 8, 8, 0, 16)))
    ptrs = (ctypes.c_void_p * 2)(16, 16)
    Lb = pkg.lib()
    assert Lb.dcnv4_forward_grouped(arr, 0, 0, ptrs, ptrs, ptrs, None) == b.ERR_INVALID_ARG
    assert Lb.dcnv4_forward_grouped(arr, 9, 0, ptrs, ptrs, ptrs, None) == b.ERR_INVALID_ARG
    assert Lb.dcnv4_forward_grouped(arr, 2, 0, None, ptrs, ptrs, None) == b.ERR_INVALID_ARG
    assert Lb.dcnv4_forward_grouped(arr, 2, 0, ptrs, ptrs, ptrs, None) == b.ERR_INVALID_ARG
    assert b"problem 1" in Lb.dcnv4_last_error()
    empty = (PP * 1)(ctypes.pointer(b.make_params(0, 8, 8, 2, 16)))
    nul = (ctypes.c_void_p * 1)(None)
    assert Lb.dcnv4_forward_grouped(empty, 1, 0, nul, nul, nul, None) == b.OK


def test_binding_rejects_bad_buffers_and_weights():
    """every caller-supplied buffer and the module weights are shape-checked in the
    binding before the ABI call (CPU tensors are rejected first, so use meta checks only)."""
    import torch
    from paper_2401_06197_b200 import module as mod
    with pytest.raises(ValueError):
        b._check_buffer(torch.empty(2, 3), (2, 4), torch.empty(1), "out")
    with pytest.raises(ValueError):
        b._check_buffer(torch.empty(2, 4, dtype=torch.float16), (2, 4), torch.empty(1), "out")
    with pytest.raises(ValueError):
        b._check_buffer(torch.empty(4, 2).t(), (2, 4), torch.empty(1), "out")
    with pytest.raises(ValueError):
        b._workspace(torch.empty(3, dtype=torch.uint8), 16, torch.empty(1))
    with pytest.raises(ValueError):
        mod._check_linear(torch.empty(108, 32), None, 4, 64, 9)
    with pytest.raises(ValueError):
        mod._check_linear(torch.empty(108, 64), torch.empty(100), 4, 64, 9)
    mod._check_linear(torch.empty(108, 64), torch.empty(108), 4, 64, 9)
