"""Pins of the module-path oracle (R21), CPU only.

oracle.offset_mask_linear is the fused offset/mask linear layer of P:334; oracle.round_to
is the fp64 -> storage-dtype rounding of reading R21; oracle.module_forward is the
lightweight module: om = linear(x), y = DCNv4(x, om).  What fixes the
expected values:
  * round_to: numpy's correctly rounded fp64 -> fp16 / fp32 casts, torch's fp32 -> bf16
    cast on fp32-exact inputs, hand-evaluated ties;
  * offset_mask_linear: torch conv2d with a 1x1 kernel (a different library routine
    than the oracle's matrix product), one-hot weights (om = a copy of feat columns);
  * module_forward: closed forms with W = 0 (the bias alone fixes om): zero offsets and
    a centre-only mask give y = x; all-ones masks give the 3x3 box filter (torch conv2d);
    an integer offset shifts x with zero fill.
A dropped bias, a transposed weight, a missing padding zero or a double rounding fails
one of them.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from tests.helpers import geom, pack_om


def test_round_to_matches_correct_casts():
    rs = np.random.default_rng(3)
    v = rs.standard_normal(100000) * np.exp(rs.uniform(-35, 12, 100000))
    with np.errstate(over="ignore"):
        assert np.array_equal(oracle.round_to(v, "f16"), v.astype(np.float16).astype(np.float64))
    assert np.array_equal(oracle.round_to(v, "f32"), v.astype(np.float32).astype(np.float64))
    # bf16: torch's fp32 -> bf16 cast is RN-even; feed fp32-exact values so no double rounding
    v32 = (rs.standard_normal(100000) * np.exp(rs.uniform(-80, 80, 100000))).astype(np.float32)
    ref = torch.from_numpy(v32).bfloat16().double().numpy()
    assert np.array_equal(oracle.round_to(v32.astype(np.float64), "bf16"), ref)


def test_round_to_ties_and_limits():
    u16 = 2.0 ** -10  # fp16 ulp at 1
    assert oracle.round_to(1 + u16 / 2, "f16") == 1.0            # tie -> even (1.0)
    assert oracle.round_to(1 + 3 * u16 / 2, "f16") == 1 + 2 * u16  # tie -> even (1+2u)
    assert oracle.round_to(1 + u16 / 2 + 1e-12, "f16") == 1 + u16
    assert oracle.round_to(2.0 ** -25, "f16") == 0.0             # half of the min subnormal
    assert oracle.round_to(3 * 2.0 ** -25, "f16") == 2.0 ** -23
    assert oracle.round_to(65519.99, "f16") == 65504.0
    assert np.isinf(oracle.round_to(65520.0, "f16"))
    u8 = 2.0 ** -7  # bf16 ulp at 1
    assert oracle.round_to(1 + u8 / 2, "bf16") == 1.0
    assert oracle.round_to(1 + 3 * u8 / 2, "bf16") == 1 + 2 * u8
    assert oracle.round_to(-(1 + 3 * u8 / 2), "bf16") == -(1 + 2 * u8)


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
def test_linear_matches_conv2d_1x1(dtype):
    rs = np.random.RandomState(7)
    N, H, W, C, J, S = 2, 5, 7, 48, 54, 64
    x = rs.uniform(-1, 1, (N, H, W, C))
    w = rs.uniform(-0.5, 0.5, (J, C))
    b = rs.uniform(-1, 1, J)
    om, exact, ab = oracle.offset_mask_linear(x.reshape(-1, C), w, b, S, dtype, with_abs=True)
    ref = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w)[:, :, None, None],
                   torch.from_numpy(b)).permute(0, 2, 3, 1).reshape(-1, J).numpy()
    np.testing.assert_allclose(exact[:, :J], ref, rtol=0, atol=1e-13)
    assert np.all(exact[:, J:] == 0) and np.all(om[:, J:] == 0) and np.all(ab[:, J:] == 0)
    # rounding: at most half an ulp of T away from the exact value
    p = {"f32": 24, "f16": 11, "bf16": 8}[dtype]
    half_ulp = np.ldexp(1.0, np.frexp(exact)[1] - p - 1)
    assert np.all(np.abs(om - exact) <= half_ulp)
    ref_ab = np.abs(x.reshape(-1, C)) @ np.abs(w).T + np.abs(b)
    np.testing.assert_allclose(ab[:, :J], ref_ab, rtol=1e-14)
    assert np.all(ab[:, :J] >= np.abs(exact[:, :J]) - 1e-12)


def test_linear_one_hot_copies_columns():
    rs = np.random.RandomState(1)
    R, C, J, S = 37, 24, 10, 16
    f = rs.uniform(-4, 4, (R, C)).astype(np.float16).astype(np.float64)  # fp16-exact
    cols = rs.randint(0, C, J)
    w = np.zeros((J, C))
    w[np.arange(J), cols] = 1.0
    om = oracle.offset_mask_linear(f, w, None, S, "f16")
    assert np.array_equal(om[:, :J], f[:, cols])
    assert np.all(om[:, J:] == 0)
    b = np.arange(J, dtype=np.float64)  # integers: exact in every dtype
    om = oracle.offset_mask_linear(f, np.zeros((J, C)), b, S, "bf16")
    assert np.array_equal(om[:, :J], np.broadcast_to(b, (R, J)))


def _bias(G, K, dx=0.0, dy=0.0, m=None):
    mm = np.zeros((1, 1, 1, G, K)) if m is None else np.broadcast_to(m, (1, 1, 1, G, K))
    return pack_om(np.full((1, 1, 1, G, K), dx), np.full((1, 1, 1, G, K), dy), mm).reshape(-1)


def test_module_bias_only_closed_forms():
    G, D, H, W = 2, 8, 6, 9
    g = geom(N=2, H=H, W=W, G=G, D=D, kh=3, kw=3, sh=1, sw=1, ph=1, pw=1, dh=1, dw=1)
    x = np.random.RandomState(4).uniform(-1, 1, (2, H, W, G * D))
    J, C = 3 * G * g.K, G * D
    w0 = np.zeros((J, C))
    centre = np.zeros(g.K)
    centre[4] = 1.0  # k = i*kh + j = 1*3 + 1: the (0, 0) tap
    y = oracle.module_forward(g, x, w0, _bias(G, g.K, m=centre))
    np.testing.assert_array_equal(y, x)
    # all masks 1, zero offsets: 3x3 box filter with zero padding
    y = oracle.module_forward(g, x, w0, _bias(G, g.K, m=np.ones(g.K)))
    box = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.ones(C, 1, 3, 3, dtype=torch.float64),
                   padding=1, groups=C).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(y, box, rtol=0, atol=1e-14)
    # dx = +1 on every point, centre mask only: y[.., w] = x[.., w + 1], zero at the right edge
    y = oracle.module_forward(g, x, w0, _bias(G, g.K, dx=1.0, m=centre))
    np.testing.assert_array_equal(y[:, :, :-1], x[:, :, 1:])
    assert np.all(y[:, :, -1] == 0)


def test_module_uses_rounded_linear_output():
    """A weight that yields a non-representable offset: the operator sees round_T(om)."""
    G, D = 1, 8
    g = geom(N=1, H=4, W=4, G=G, D=D, kh=3, kw=3, sh=1, sw=1, ph=1, pw=1, dh=1, dw=1)
    x = np.random.RandomState(5).uniform(-1, 1, (1, 4, 4, D))
    J = 3 * G * g.K
    w = np.zeros((J, D))
    w[0, 0] = 1.0 / 3.0  # dx_0 = x[.., 0] / 3
    b = _bias(G, g.K, m=np.ones(g.K))
    y, _, om = oracle.module_forward(g, x, w, b, "bf16", with_abs=True)
    want = oracle.round_to(x[..., 0] / 3.0, "bf16")
    np.testing.assert_array_equal(om[..., 0], want)
    np.testing.assert_array_equal(y, oracle.forward(g, x, om))
