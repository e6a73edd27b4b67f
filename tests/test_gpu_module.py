"""GPU parity of the module path (include/dcnv4_module.h) against the
fp64 oracle (oracle.offset_mask_linear / oracle.module_forward, reading R21).

offset_mask: every element within the rigorous bound of an fp32-accumulated, once-rounded
result, |om - exact| <= E + half_ulp_T(|exact| + E) with E = (C_in + 1) * 2^-24 * A
(A = sum_c |x_c w_jc| + |b_j|, the products of two halves being exact in fp32), and
>= 99% of elements bit-equal to the oracle's RN_T(exact); padding columns exactly 0.
Module forward y: abs-scaled error <= 1e-2 (north_star's half-precision bar).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2401_06197_b200 import module

pytestmark = pytest.mark.gpu

P_BITS = {"f16": 11, "bf16": 8}

# (N, H, W, G, D, om_stride or None, bias?)
CASES = [
    (1, 8, 8, 4, 16, None, True),     # C=64, J=108 -> S=112: one 128x128 tile, clipped cols
    (2, 7, 9, 4, 16, 128, True),      # ragged rows (126), S > J padding
    (2, 14, 14, 8, 16, None, True),   # C=128, J=216 -> S=224
    (1, 14, 14, 16, 16, None, False),  # C=256, J=432 (two column tiles), no bias
    (1, 7, 7, 32, 16, None, True),    # C=512, J=864 (four column tiles, 8 k blocks)
    (1, 5, 6, 9, 8, None, True),      # C=72: k tail (zero-filled by TMA), J=243 -> S=248
    (1, 8, 8, 80, 16, None, True),    # C=1280 (U-Net stage 3), J=2160, nine column tiles
    (3, 56, 56, 4, 16, None, True),   # c2 stage 1 geometry, 9408 rows (74 row tiles)
]


def _run(case, dt, dev):
    N, H, W, G, D, S, with_bias = case
    C, K = G * D, 9
    x, _, _ = synth.make_case(N, H, W, G, D, H, W, K, 3 * G * K, dt, with_gy=False)
    w, b = synth.make_linear(C, G, K, dt, seed=N * 1000 + C)
    b = b if with_bias else None
    S = S or module.om_stride_for(G, K)
    om = module.offset_mask_linear(x.to(dev), w.to(dev), b.to(dev) if b is not None else None, G,
                                   om_stride=S)
    torch.cuda.synchronize()
    return x, w, b, S, om.cpu()


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}x{c[2]}xG{c[3]}D{c[4]}" for c in CASES])
def test_offset_mask_linear(case, dt, cuda_device):
    x, w, b, S, om = _run(case, dt, cuda_device)
    C = x.shape[-1]
    J = w.shape[0]
    ref, exact, ab = oracle.offset_mask_linear(x.reshape(-1, C), w, b, S, dt, with_abs=True)
    got = om.reshape(-1, S).double().numpy()
    assert np.all(got[:, J:] == 0)
    E = (C + 1) * 2.0 ** -24 * ab
    half_ulp = np.ldexp(1.0, np.frexp(np.abs(exact) + E)[1] - P_BITS[dt] - 1)
    err = np.abs(got - exact)
    bad = err > E + half_ulp
    assert not bad.any(), f"{bad.sum()} elements outside the bound, worst {err[bad].max()}"
    assert np.mean(got == ref) >= 0.99


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("case", [CASES[0], CASES[1], CASES[4]], ids=["c64", "ragged", "c512"])
def test_module_forward(case, dt, cuda_device):
    N, H, W, G, D, S, with_bias = case
    C, K = G * D, 9
    x, _, _ = synth.make_case(N, H, W, G, D, H, W, K, 3 * G * K, dt, with_gy=False)
    w, b = synth.make_linear(C, G, K, dt, seed=7)
    S = S or module.om_stride_for(G, K)
    y = module.module_forward(x.to(cuda_device), w.to(cuda_device), b.to(cuda_device), G,
                              om_stride=S)
    torch.cuda.synchronize()
    g = oracle.Geometry(N=N, H=H, W=W, G=G, D=D, om_stride=S)
    ref, ra, _ = oracle.module_forward(g, x, w, b, dt, with_abs=True)
    assert oracle.abs_scaled_error(y.cpu(), ref, ra) <= 1e-2


def test_f32_unsupported(cuda_device):
    x = torch.zeros((1, 4, 4, 64), device=cuda_device)
    w = torch.zeros((108, 64), device=cuda_device)
    with pytest.raises(Exception, match="UNSUPPORTED"):
        module.offset_mask_linear(x, w, None, 4)


# ---------------------------------------------------------------- fused module forward
# (N, H, W, G, D, offset_scale, softmax, bias?)
FUSED = [
    (1, 8, 8, 4, 16, 1.0, False, True),     # one ragged tile (8 of 16 rows)
    (2, 7, 9, 4, 16, 1.0, False, True),     # ragged rows and columns
    (1, 20, 13, 8, 16, 1.0, False, True),   # C=128: 2 group blocks, 2 k blocks
    (1, 14, 14, 16, 16, 1.0, False, False),  # C=256: 4 k blocks (ring reuse), no bias
    (1, 7, 7, 32, 16, 1.0, False, True),    # C=512: 8 k blocks, 8 group blocks
    (1, 12, 10, 4, 32, 1.0, False, True),   # D=32: 2 groups per CTA
    (1, 9, 11, 2, 64, 1.0, False, True),    # D=64: 1 group per CTA
    (1, 10, 12, 12, 16, 0.5, False, True),  # C=192, offset_scale 0.5 (non-unit path)
    (1, 9, 9, 4, 16, 1.0, True, True),      # DCNv3 softmax mode
    (2, 56, 56, 4, 16, 1.0, False, True),   # c2 stage-1 geometry
]


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("case", FUSED, ids=[f"{c[0]}x{c[1]}x{c[2]}G{c[3]}D{c[4]}s{c[5]}{'sm' if c[6] else ''}"
                                             for c in FUSED])
def test_fused_module_forward(case, dt, cuda_device):
    N, H, W, G, D, s, sm, with_bias = case
    C, K = G * D, 9
    x, _, _ = synth.make_case(N, H, W, G, D, H, W, K, 3 * G * K, dt, with_gy=False)
    w, b = synth.make_linear(C, G, K, dt, seed=11)
    b = b if with_bias else None
    xd, wd = x.to(cuda_device), w.to(cuda_device)
    bd = b.to(cuda_device) if b is not None else None
    y = module.forward_fused(xd, wd, bd, G, offset_scale=s, softmax=sm)
    # the two-call path (linear kernel + dcnv4_forward) computes the same function
    om = module.offset_mask_linear(xd, wd, bd, G)
    from paper_2401_06197_b200 import binding
    y2 = binding.forward(xd, om, G, 3, 1, 1, 1, s, softmax=sm)
    torch.cuda.synchronize()
    g = oracle.Geometry(N=N, H=H, W=W, G=G, D=D, offset_scale=s, softmax=sm)
    ref, ra, _ = oracle.module_forward(g, x, w, b, dt, with_abs=True)
    err = oracle.abs_scaled_error(y.cpu(), ref, ra)
    assert err <= 1e-2, err
    assert oracle.abs_scaled_error(y2.cpu(), ref, ra) <= 1e-2
    # same function: the two paths differ only by the linear's fp32 summation order (om
    # rounding flips) and, where dcnv4_forward takes its global-gather kernel, fp32 vs
    # FHFMA weights (R10)
    assert oracle.abs_scaled_error(y.cpu(), y2.cpu(), ra) <= 1e-2


def test_fused_deterministic_and_unsupported(cuda_device):
    x, _, _ = synth.make_case(1, 16, 16, 8, 16, 16, 16, 9, 216, "bf16", with_gy=False)
    w, b = synth.make_linear(128, 8, 9, "bf16")
    xd, wd, bd = x.to(cuda_device), w.to(cuda_device), b.to(cuda_device)
    y1 = module.forward_fused(xd, wd, bd, 8)
    y2 = module.forward_fused(xd, wd, bd, 8)
    assert torch.equal(y1, y2)
    with pytest.raises(Exception, match="UNSUPPORTED"):
        module.forward_fused(xd.float(), wd.float(), bd.float(), 8)
    with pytest.raises(Exception, match="UNSUPPORTED"):  # D = 8 halves = 16 B
        module.forward_fused(xd, torch.zeros((27 * 16, 128), dtype=xd.dtype, device=cuda_device), None, 16)
