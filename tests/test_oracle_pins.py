"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names what fixes the expected value:
  * library routines: torch conv2d (zero offsets) and grid_sample + autograd (general);
  * closed forms and hand-evaluated examples;
  * algebraic invariants (linearity, adjoint, Euler, translation equivariance);
  * exact finite differences (the operator is piecewise linear in the offsets).
A plausible slip in the oracle -- a dropped term, a swapped (dx, dy), a wrong tap order,
an off-by-one in padding or output size, a wrong offset_scale reading -- fails one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from tests.helpers import geom, pack_om, rng_case, unpack_om

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

# (kh, kw, sh, sw, ph, pw, dh, dw) variants: stride 1/2, pad 0/1/2, dilation 1/2,
# kernels 1x1, 3x3, 5x5, 3x5 and an even 2x2 (reading R15).
GEOMS = [
    (3, 3, 1, 1, 1, 1, 1, 1),
    (3, 3, 2, 2, 1, 1, 1, 1),
    (3, 3, 1, 1, 2, 2, 2, 2),
    (3, 3, 2, 1, 0, 1, 1, 1),
    (1, 1, 1, 1, 0, 0, 1, 1),
    (5, 5, 1, 1, 2, 2, 1, 1),
    (3, 5, 1, 2, 1, 2, 1, 2),
    (2, 2, 1, 1, 0, 1, 1, 1),
]


def _g(N, H, W, G, D, v, s=1.0, S=0, softmax=False):
    kh, kw, sh, sw, ph, pw, dh, dw = v
    return geom(N=N, H=H, W=W, G=G, D=D, kh=kh, kw=kw, sh=sh, sw=sw, ph=ph, pw=pw, dh=dh,
                dw=dw, offset_scale=s, om_stride=S, softmax=softmax)


def _conv_weight(m_gk, g: oracle.Geometry):
    """Depthwise conv2d weight w[c, 0, j, i] = m[g(c), i*kh + j] (reading R2)."""
    w = np.zeros((g.C, 1, g.kh, g.kw))
    for c in range(g.C):
        for i in range(g.kw):
            for j in range(g.kh):
                w[c, 0, j, i] = m_gk[c // g.D, i * g.kh + j]
    return torch.from_numpy(w)


def _conv2d(x, w, g):
    xt = torch.from_numpy(x).permute(0, 3, 1, 2)
    y = F.conv2d(xt, w, stride=(g.sh, g.sw), padding=(g.ph, g.pw), dilation=(g.dh, g.dw),
                 groups=g.C)
    return y.permute(0, 2, 3, 1).numpy()


# ---------------------------------------------------------------- library reductions
@pytest.mark.parametrize("v", GEOMS)
def test_zero_offset_reduces_to_depthwise_conv2d(v):
    """P:197 "as in regular convolutions": dp = 0 and location-independent m
    => y = depthwise conv2d (cross-correlation) with taps m_gk.  Pins the output
    size, the tap order (x-outer), the zero padding, stride and dilation."""
    g = _g(2, 9, 11, 2, 3, v)
    rs = np.random.RandomState(1)
    Ho, Wo = g.out_hw()
    x = rs.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    m_gk = rs.uniform(-1, 1, (g.G, g.K))
    m = np.broadcast_to(m_gk, (g.N, Ho, Wo, g.G, g.K))
    z = np.zeros_like(m)
    y = oracle.forward(g, x, pack_om(z, z, m))
    ref = _conv2d(x, _conv_weight(m_gk, g), g)
    assert y.shape == ref.shape
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-13)


def test_offset_scale_two_is_dilation_two():
    """Reading R5 (p = p0 + s*(p_k + dp)): with dp = 0 and s = 2 a 3x3 dilation-1
    window becomes conv2d with dilation 2 and padding ph + 1 (same centre)."""
    g = _g(1, 10, 9, 2, 2, (3, 3, 1, 1, 1, 1, 1, 1), s=2.0)
    rs = np.random.RandomState(2)
    x = rs.uniform(-1, 1, (1, 10, 9, 4))
    m_gk = rs.uniform(-1, 1, (2, 9))
    Ho, Wo = g.out_hw()
    m = np.broadcast_to(m_gk, (1, Ho, Wo, 2, 9))
    z = np.zeros_like(m)
    y = oracle.forward(g, x, pack_om(z, z, m))
    g2 = _g(1, 10, 9, 2, 2, (3, 3, 1, 1, 2, 2, 2, 2))
    ref = _conv2d(x, _conv_weight(m_gk, g2), g2)
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-13)


def test_offset_scale_half_is_midpoint_kernel():
    """s = 0.5, dp = 0: taps sit at centre +-0.5, i.e. the bilinear midpoint of two
    pixels.  The equivalent 3x3 kernel is sum_ij m_ij A_j (x) A_i with
    A_0 = [.5,.5,0], A_1 = [0,1,0], A_2 = [0,.5,.5] (hand derivation)."""
    g = _g(1, 8, 7, 1, 3, (3, 3, 1, 1, 1, 1, 1, 1), s=0.5)
    rs = np.random.RandomState(3)
    x = rs.uniform(-1, 1, (1, 8, 7, 3))
    m_gk = rs.uniform(-1, 1, (1, 9))
    A = np.array([[.5, .5, 0], [0, 1, 0], [0, .5, .5]])
    weff = np.zeros((3, 3))
    for i in range(3):
        for j in range(3):
            weff += m_gk[0, i * 3 + j] * np.outer(A[j], A[i])
    w = torch.from_numpy(np.broadcast_to(weff, (3, 1, 3, 3)).copy())
    Ho, Wo = g.out_hw()
    m = np.broadcast_to(m_gk, (1, Ho, Wo, 1, 9))
    z = np.zeros_like(m)
    y = oracle.forward(g, x, pack_om(z, z, m))
    ref = _conv2d(x, w, g)
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-13)


def _grid_sample_model(g: oracle.Geometry, x, dx, dy, m):
    """y = sum_k m_k * grid_sample(x_g, loc_k) with torch autograd (independent
    bilinear / zero-padding / backward implementation)."""
    Ho, Wo = g.out_hw()
    cy = g.dh * (g.kh - 1) // 2
    cx = g.dw * (g.kw - 1) // 2
    ho = torch.arange(Ho, dtype=torch.float64).view(1, Ho, 1)
    wo = torch.arange(Wo, dtype=torch.float64).view(1, 1, Wo)
    ys = []
    for grp in range(g.G):
        xg = x[..., grp * g.D:(grp + 1) * g.D].permute(0, 3, 1, 2)
        acc = 0
        for i in range(g.kw):
            for j in range(g.kh):
                k = i * g.kh + j
                py = (ho * g.sh - g.ph + cy) + g.offset_scale * ((j * g.dh - cy) + dy[..., grp, k])
                px = (wo * g.sw - g.pw + cx) + g.offset_scale * ((i * g.dw - cx) + dx[..., grp, k])
                grid = torch.stack([(2 * px + 1) / g.W - 1, (2 * py + 1) / g.H - 1], -1)
                smp = F.grid_sample(xg, grid, mode="bilinear", padding_mode="zeros",
                                    align_corners=False)
                acc = acc + m[..., grp, k].unsqueeze(1) * smp
        ys.append(acc.permute(0, 2, 3, 1))
    return torch.cat(ys, -1)


@pytest.mark.parametrize("v,s", [(GEOMS[0], 1.0), (GEOMS[1], 0.5), (GEOMS[2], 2.0),
                                 (GEOMS[3], 1.0), (GEOMS[5], 1.0), (GEOMS[6], 0.5),
                                 (GEOMS[7], 1.0)])
def test_grid_sample_equivalence_forward_and_backward(v, s):
    """Forward vs torch grid_sample (align_corners=False, zeros padding) and all three
    gradients vs torch autograd through it."""
    g = _g(2, 7, 8, 2, 3, v, s=s, S=3 * 2 * v[0] * v[1] + 5)
    x, om, gy = rng_case(4, g)
    om[..., 3 * g.G * g.K:] = 7.0  # padding channels must be ignored
    dx, dy, m = (torch.tensor(a, requires_grad=True) for a in unpack_om(om, g.G, g.K))
    xt = torch.tensor(x, requires_grad=True)
    yt = _grid_sample_model(g, xt, dx, dy, m)
    (yt * torch.from_numpy(gy)).sum().backward()
    y = oracle.forward(g, x, om)
    gx, gom = oracle.backward(g, x, om, gy)
    np.testing.assert_allclose(y, yt.detach().numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(gx, xt.grad.numpy(), rtol=0, atol=1e-12)
    gdx, gdy, gm = unpack_om(gom, g.G, g.K)
    np.testing.assert_allclose(gm, m.grad.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(gdx, dx.grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(gdy, dy.grad.numpy(), rtol=0, atol=1e-11)
    assert np.all(gom[..., 3 * g.G * g.K:] == 0.0)


# ---------------------------------------------------------------- closed forms
def test_spec_bilinear_examples_golden():
    """SPEC S:122-124 via a 1x1 kernel (K=1, pad 0): the sample sits at (ho+dy, wo+dx)."""
    with open(os.path.join(GOLDEN, "spec_bilinear.json")) as f:
        fx = json.load(f)
    plane = np.array(fx["plane"], np.float64)
    H, W = plane.shape
    g = _g(1, H, W, 1, 1, (1, 1, 1, 1, 0, 0, 1, 1))
    for case in fx["cases"]:
        ho, wo = case["output"]
        py, px = case["point"]
        dy = np.zeros((1, H, W, 1, 1))
        dx = np.zeros((1, H, W, 1, 1))
        dy[0, ho, wo, 0, 0] = py - ho
        dx[0, ho, wo, 0, 0] = px - wo
        m = np.ones((1, H, W, 1, 1))
        y = oracle.forward(g, plane.reshape(1, H, W, 1), pack_om(dx, dy, m))
        assert y[0, ho, wo, 0] == case["value"], case


def test_identity_1x1():
    """K=1, dp=0, m=1 => y == x exactly and grad_x == grad_y."""
    g = _g(2, 5, 6, 3, 2, (1, 1, 1, 1, 0, 0, 1, 1))
    rs = np.random.RandomState(5)
    x = rs.uniform(-1, 1, (2, 5, 6, 6))
    gy = rs.uniform(-1, 1, (2, 5, 6, 6))
    z = np.zeros((2, 5, 6, 3, 1))
    om = pack_om(z, z, np.ones_like(z))
    assert np.array_equal(oracle.forward(g, x, om), x)
    gx, _ = oracle.backward(g, x, om, gy)
    assert np.array_equal(gx, gy)


def test_pure_shift_orders_dx_before_dy():
    """Reading R2: channel 2k is dx (along W), 2k+1 is dy (along H).  Centre tap only
    (k = 4 for 3x3), dx = +1 => y[h, w] = x[h, w+1]; dy = +1 => y[h, w] = x[h+1, w]."""
    g = _g(1, 6, 7, 1, 2, GEOMS[0])
    rs = np.random.RandomState(6)
    x = rs.uniform(-1, 1, (1, 6, 7, 2))
    z = np.zeros((1, 6, 7, 1, 9))
    m = z.copy()
    m[..., 4] = 1.0
    one = z.copy()
    one[..., 4] = 1.0
    y = oracle.forward(g, x, pack_om(one, z, m))
    ref = np.zeros_like(x)
    ref[:, :, :-1] = x[:, :, 1:]
    assert np.array_equal(y, ref)
    y = oracle.forward(g, x, pack_om(z, one, m))
    ref = np.zeros_like(x)
    ref[:, :-1] = x[:, 1:]
    assert np.array_equal(y, ref)


def test_tap_order_on_ramp():
    """Reading R2 by hand: on the ramp x = 100*h + w, point k = i*kh + j samples
    (h - 1 + j, w - 1 + i) at zero offset (3x3, pad 1).  Point k=1 (i=0, j=1) is
    (h, w-1); point k=3 (i=1, j=0) is (h-1, w)."""
    g = _g(1, 5, 5, 1, 1, GEOMS[0])
    hh, ww = np.meshgrid(np.arange(5.0), np.arange(5.0), indexing="ij")
    x = (100 * hh + ww).reshape(1, 5, 5, 1)
    z = np.zeros((1, 5, 5, 1, 9))
    for k, (dh_, dw_) in [(1, (0, -1)), (3, (-1, 0)), (0, (-1, -1)), (8, (1, 1)), (2, (1, -1))]:
        m = z.copy()
        m[..., k] = 1.0
        y = oracle.forward(g, x, pack_om(z, z, m))
        assert y[0, 2, 2, 0] == 100 * (2 + dh_) + (2 + dw_), k


@pytest.mark.parametrize("s", [0.5, 1.0, 2.0])
def test_affine_ramp_closed_form(s):
    """x(h, w, c) = a*h + b*w + kappa_c with every corner in bounds:
    y = sum_k m_k (a*py_k + b*px_k + kappa_c) where (py_k, px_k) is the exact location;
    grad_dy_k = s*m_k*a*sum_c gy_c, grad_dx_k = s*m_k*b*sum_c gy_c, even at kinks.
    The location is checked independently by evaluating the ramp at the sampled point
    derived from pure-shift semantics (offsets add to the tap position, scaled by s)."""
    H = W = 12
    g = _g(1, H, W, 2, 3, GEOMS[0], s=s)
    a, b = 0.7, -1.3
    kappa = np.array([0.25, -2.0, 1.5, 0.5, 3.0, -1.0])
    hh, ww = np.meshgrid(np.arange(H, dtype=float), np.arange(W, dtype=float), indexing="ij")
    x = (a * hh[..., None] + b * ww[..., None] + kappa).reshape(1, H, W, 6)
    rs = np.random.RandomState(7)
    dx = rs.uniform(-0.4, 0.4, (1, H, W, 2, 9))
    dy = rs.uniform(-0.4, 0.4, (1, H, W, 2, 9))
    dx[0, 5, 5, 0, :] = 0.0  # exact kinks (integer coordinates at s = 1)
    dy[0, 5, 5, 0, :] = 0.0
    m = rs.uniform(-1, 1, (1, H, W, 2, 9))
    gy = rs.uniform(-1, 1, (1, H, W, 6))
    om = pack_om(dx, dy, m)
    y = oracle.forward(g, x, om)
    _, gom = oracle.backward(g, x, om, gy)
    gdx, gdy, _ = unpack_om(gom, 2, 9)
    # the sampled location of tap (i, j): centre (h, w) + s*((j-1) + dy, (i-1) + dx)
    j = np.tile(np.arange(3), 3)
    i = np.repeat(np.arange(3), 3)
    for h in range(3, 9):  # interior: |s*(1 + 0.4)| <= 2.8 < 3 keeps corners in bounds
        for w in range(3, 9):
            for grp in range(2):
                py = h + s * ((j - 1) + dy[0, h, w, grp])
                px = w + s * ((i - 1) + dx[0, h, w, grp])
                mk = m[0, h, w, grp]
                for c in range(3):
                    ref = np.sum(mk * (a * py + b * px + kappa[grp * 3 + c]))
                    assert abs(y[0, h, w, grp * 3 + c] - ref) < 1e-12
                sg = gy[0, h, w, grp * 3:(grp + 1) * 3].sum()
                np.testing.assert_allclose(gdy[0, h, w, grp], s * mk * a * sg, atol=1e-12)
                np.testing.assert_allclose(gdx[0, h, w, grp], s * mk * b * sg, atol=1e-12)


def test_constant_input_partition_of_unity():
    """x == kappa with all corners in bounds: y = kappa * sum_k m_k, grad_offset = 0."""
    H = W = 10
    g = _g(1, H, W, 2, 2, GEOMS[0])
    x = np.full((1, H, W, 4), 1.75)
    rs = np.random.RandomState(8)
    dx = rs.uniform(-0.9, 0.9, (1, H, W, 2, 9))
    dy = rs.uniform(-0.9, 0.9, (1, H, W, 2, 9))
    m = rs.uniform(-1, 1, (1, H, W, 2, 9))
    om = pack_om(dx, dy, m)
    y = oracle.forward(g, x, om)
    _, gom = oracle.backward(g, x, om, rs.uniform(-1, 1, (1, H, W, 4)))
    gdx, gdy, _ = unpack_om(gom, 2, 9)
    sl = (0, slice(2, 8), slice(2, 8))
    ref = 1.75 * m.sum(-1)
    np.testing.assert_allclose(y[sl].reshape(6, 6, 2, 2), np.repeat(ref[sl][..., None], 2, -1),
                               atol=1e-13)
    assert np.abs(gdx[sl]).max() < 1e-13 and np.abs(gdy[sl]).max() < 1e-13


def test_all_samples_out_of_bounds():
    """dp = +3H pushes every sample outside: y = 0, grad_m = 0, grad_dp = 0, grad_x = 0."""
    g = _g(1, 5, 5, 2, 2, GEOMS[0])
    rs = np.random.RandomState(9)
    x = rs.uniform(-1, 1, (1, 5, 5, 4))
    big = np.full((1, 5, 5, 2, 9), 15.0)
    om = pack_om(big, -big, rs.uniform(-1, 1, (1, 5, 5, 2, 9)))
    y = oracle.forward(g, x, om)
    gx, gom = oracle.backward(g, x, om, rs.uniform(-1, 1, (1, 5, 5, 4)))
    assert not y.any() and not gx.any() and not gom.any()


def test_bilinear_border_corner_zero_padding():
    """Per-corner zero padding (reading R6): a sample at (-0.5, 0) on a plane of ones
    sees one in-bounds corner row with weight 0.5 => 0.5."""
    g = _g(1, 3, 3, 1, 1, (1, 1, 1, 1, 0, 0, 1, 1))
    x = np.ones((1, 3, 3, 1))
    dy = np.zeros((1, 3, 3, 1, 1))
    dy[0, 0, 0] = -0.5
    om = pack_om(np.zeros_like(dy), dy, np.ones_like(dy))
    assert oracle.forward(g, x, om)[0, 0, 0, 0] == 0.5


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("v", GEOMS[:4])
def test_linearity_adjoint_euler(v):
    """Linear in x and in m; grad_x is the adjoint of x -> y:
    <gy, F(x)> = <grad_x, x>; Euler in m: sum m_k grad_m_k = <gy, y>."""
    g = _g(2, 7, 6, 2, 3, v)
    x, om, gy = rng_case(10, g)
    x2, om2, _ = rng_case(11, g)
    y = oracle.forward(g, x, om)
    np.testing.assert_allclose(oracle.forward(g, 2.0 * x - 3.0 * x2, om),
                               2.0 * y - 3.0 * oracle.forward(g, x2, om), atol=1e-12)
    dx, dy, m = unpack_om(om, g.G, g.K)
    _, _, m2 = unpack_om(om2, g.G, g.K)
    ya = oracle.forward(g, x, pack_om(dx, dy, m + 0.5 * m2))
    yb = oracle.forward(g, x, pack_om(dx, dy, m2))
    np.testing.assert_allclose(ya, y + 0.5 * yb, atol=1e-12)
    gx, gom = oracle.backward(g, x, om, gy)
    np.testing.assert_allclose(np.sum(gy * y), np.sum(gx * x), rtol=1e-12)
    _, _, gm = unpack_om(gom, g.G, g.K)
    np.testing.assert_allclose(np.sum(m * gm), np.sum(gy * y), rtol=1e-12)


def test_translation_equivariance_zero_offsets():
    """dp = 0 and location-independent m; shifting x by one pixel shifts y
    on the interior."""
    g = _g(1, 9, 9, 2, 2, GEOMS[0])
    rs = np.random.RandomState(12)
    x = rs.uniform(-1, 1, (1, 9, 9, 4))
    m = np.broadcast_to(rs.uniform(-1, 1, (2, 9)), (1, 9, 9, 2, 9))
    z = np.zeros_like(m)
    om = pack_om(z, z, m)
    y = oracle.forward(g, x, om)
    ys = oracle.forward(g, np.roll(x, 1, axis=2), om)
    np.testing.assert_allclose(ys[:, 2:-2, 3:-2], y[:, 2:-2, 2:-3], atol=1e-14)


# ---------------------------------------------------------------- finite differences
FD_CASES = [(GEOMS[0], 1.0, 1), (GEOMS[1], 0.5, 2), (GEOMS[2], 2.0, 1), (GEOMS[3], 1.0, 4),
            (GEOMS[5], 1.0, 1), (GEOMS[6], 0.5, 2), (GEOMS[4], 2.0, 2)]


@pytest.mark.parametrize("v,s,G", FD_CASES)
def test_finite_differences(v, s, G):
    """Central differences of L = <gy, y>: exact for x and m (linear) and for the
    offsets away from kinks (piecewise linear); coordinates within 2h|s| of an
    integer are skipped (after SPEC S:147)."""
    g = _g(1, 5, 6, G, 2, v, s=s)
    x, om, gy = rng_case(13 + G, g)
    gx, gom = oracle.backward(g, x, om, gy)

    def L(xx, oo):
        return float(np.sum(gy * oracle.forward(g, xx, oo)))

    h = 1e-3
    fdx = np.zeros_like(x)
    for idx in itertools.product(*map(range, x.shape)):
        xp = x.copy(); xp[idx] += h
        xm = x.copy(); xm[idx] -= h
        fdx[idx] = (L(xp, om) - L(xm, om)) / (2 * h)
    np.testing.assert_allclose(fdx, gx, rtol=0, atol=1e-9)

    Ho, Wo = g.out_hw()
    K = g.K
    cy, cx = g.dh * (g.kh - 1) // 2, g.dw * (g.kw - 1) // 2
    checked = 0
    for n, ho, wo, c in itertools.product(range(1), range(Ho), range(Wo), range(3 * G * K)):
        grp, q = divmod(c, 3 * K)
        if q < 2 * K:  # an offset channel: skip near a kink of its coordinate
            k, axis = divmod(q, 2)
            i, j = divmod(k, g.kh)
            if axis == 0:
                coord = (wo * g.sw - g.pw + cx) + s * ((i * g.dw - cx) + om[n, ho, wo, c])
            else:
                coord = (ho * g.sh - g.ph + cy) + s * ((j * g.dh - cy) + om[n, ho, wo, c])
            if abs(coord - np.round(coord)) < 2 * h * abs(s) + 1e-9:
                continue
        op = om.copy(); op[n, ho, wo, c] += h
        omm = om.copy(); omm[n, ho, wo, c] -= h
        fd = (L(x, op) - L(x, omm)) / (2 * h)
        assert abs(fd - gom[n, ho, wo, c]) < 1e-9, (ho, wo, c, fd, gom[n, ho, wo, c])
        checked += 1
    assert checked > 0.9 * Ho * Wo * 3 * G * K


def test_right_derivative_at_kinks():
    """Reading R8: at dp = 0 (s = 1) every coordinate is an integer; the one-sided
    forward difference with 0 < h < 1 equals the oracle's offset gradient exactly."""
    g = _g(1, 5, 5, 1, 2, GEOMS[0])
    rs = np.random.RandomState(20)
    x = rs.uniform(-1, 1, (1, 5, 5, 2))
    gy = rs.uniform(-1, 1, (1, 5, 5, 2))
    z = np.zeros((1, 5, 5, 1, 9))
    om = pack_om(z, z, rs.uniform(-1, 1, (1, 5, 5, 1, 9)))
    _, gom = oracle.backward(g, x, om, gy)
    h = 0.25
    for c in range(18):
        for ho, wo in [(0, 0), (2, 3), (4, 4)]:
            op = om.copy(); op[0, ho, wo, c] += h
            fd = (np.sum(gy * oracle.forward(g, x, op)) - np.sum(gy * oracle.forward(g, x, om))) / h
            assert abs(fd - gom[0, ho, wo, c]) < 1e-12


# ---------------------------------------------------------------- DCNv3 softmax mode
def test_softmax_examples_spec():
    """equal logits => 1/K each; logits (1,2,3) with K=3 =>
    (0.09003057, 0.24472847, 0.66524096).  Read the weights off with one-hot inputs."""
    g = _g(1, 1, 3, 1, 1, (1, 3, 1, 1, 0, 1, 1, 1), softmax=True)  # 1x3 kernel, pad (0,1)
    z = np.zeros((1, 1, 3, 1, 3))
    logits = z.copy()
    logits[0, 0, 1, 0] = [1.0, 2.0, 3.0]
    om = pack_om(z, z, logits)
    ref = [0.09003057, 0.24472847, 0.66524096]
    for t in range(3):
        x = np.zeros((1, 1, 3, 1))
        x[0, 0, t, 0] = 1.0  # tap i samples column wo - 1 + i
        assert abs(oracle.forward(g, x, om)[0, 0, 1, 0] - ref[t]) < 5e-9
    g9 = _g(1, 4, 4, 1, 1, GEOMS[0], softmax=True)
    x = np.random.RandomState(21).uniform(-1, 1, (1, 4, 4, 1))
    om9 = pack_om(np.zeros((1, 4, 4, 1, 9)), np.zeros((1, 4, 4, 1, 9)), np.full((1, 4, 4, 1, 9), 3.3))
    box = np.zeros_like(x)
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1), (0, 0)))
    for h in range(4):
        for w in range(4):
            box[0, h, w] = xp[0, h:h + 3, w:w + 3].sum(axis=(0, 1)) / 9.0
    np.testing.assert_allclose(oracle.forward(g9, x, om9), box, atol=1e-14)


def test_softmax_backward_finite_differences():
    g = _g(1, 4, 5, 2, 2, GEOMS[0], softmax=True)
    x, om, gy = rng_case(22, g)
    _, gom = oracle.backward(g, x, om, gy)
    h = 1e-5
    for c in list(range(18, 27)) + list(range(45, 54)):
        for ho, wo in [(0, 0), (1, 3), (3, 4)]:
            op = om.copy(); op[0, ho, wo, c] += h
            omm = om.copy(); omm[0, ho, wo, c] -= h
            fd = (np.sum(gy * oracle.forward(g, x, op)) - np.sum(gy * oracle.forward(g, x, omm))) / (2 * h)
            assert abs(fd - gom[0, ho, wo, c]) < 1e-8


def test_abs_scales_bound_values():
    """The magnitude scales dominate the values (|y| <= y_abs etc.) and are exact
    for non-negative data (x >= 0, m >= 0, gy >= 0 => scale == value for y, gx, gm)."""
    g = _g(1, 6, 6, 2, 2, GEOMS[0])
    x, om, gy = rng_case(23, g)
    y, ya = oracle.forward(g, x, om, with_abs=True)
    gx, gom, gxa, goma = oracle.backward(g, x, om, gy, with_abs=True)
    assert np.all(np.abs(y) <= ya + 1e-15) and np.all(np.abs(gx) <= gxa + 1e-15)
    assert np.all(np.abs(gom) <= goma + 1e-15)
    dx, dy, m = unpack_om(om, 2, 9)
    omp = pack_om(dx, dy, np.abs(m))
    y, ya = oracle.forward(g, np.abs(x), omp, with_abs=True)
    np.testing.assert_allclose(y, ya, atol=1e-14)
    gx, gom, gxa, goma = oracle.backward(g, np.abs(x), omp, np.abs(gy), with_abs=True)
    np.testing.assert_allclose(gx, gxa, atol=1e-14)
    np.testing.assert_allclose(unpack_om(gom, 2, 9)[2], unpack_om(goma, 2, 9)[2], atol=1e-14)


def test_thread_count_independence():
    """the oracle result does not depend on the OpenMP thread count."""
    import subprocess
    import sys
    code = ("import numpy as np, oracle; from tests.helpers import geom, rng_case;"
            "g = geom(N=3, H=6, W=7, G=4, D=2); x, om, gy = rng_case(30, g);"
            "y = oracle.forward(g, x, om); gx, gom = oracle.backward(g, x, om, gy);"
            "print(hash((y.tobytes(), gx.tobytes(), gom.tobytes())))")
    root = os.path.dirname(GOLDEN)[:-len("/tests")]
    outs = set()
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONHASHSEED="0")
        outs.add(subprocess.check_output([sys.executable, "-c", code], cwd=root, env=env).strip())
    assert len(outs) == 1


# ------------------------------------------------- magnitude scales: equality cases
def _aim_offsets(g, ty, tx):
    """Offsets that put sample (pixel, group, tap) at (ty, tx) [N,Ho,Wo,G,K] under the
    convention sheet (readings R2/R4/R5):
    py = (ho*sh - ph + cy) + s*(j*dh - cy + dy)."""
    Ho, Wo = g.out_hw()
    cy, cx = (g.dh * (g.kh - 1)) // 2, (g.dw * (g.kw - 1)) // 2
    ho = np.arange(Ho).reshape(1, Ho, 1, 1, 1)
    wo = np.arange(Wo).reshape(1, 1, Wo, 1, 1)
    k = np.arange(g.K).reshape(1, 1, 1, 1, g.K)
    i, j = k // g.kh, k % g.kh
    dy = (ty - (ho * g.sh - g.ph + cy)) / g.offset_scale - (j * g.dh - cy)
    dx = (tx - (wo * g.sw - g.pw + cx)) / g.offset_scale - (i * g.dw - cx)
    return dx, dy


@pytest.mark.parametrize("s,softmax", [(1.0, False), (0.5, False), (2.0, False), (1.0, True)])
@pytest.mark.parametrize("axis", ["y", "x"])
def test_offset_grad_scale_equals_value_when_terms_agree(s, softmax, axis):
    """the offset-gradient scale is |s m| sum_c |gy_c| sum_corner |dw| |X|.
    When every term of grad_d = s m sum_c gy_c sum_corner dw X has the same sign, the
    scale equals |grad_d| exactly.  For d/dy the corner derivatives are -(1-fx), -fx on
    the top row and +(1-fx), +fx on the bottom row, so: every sample between rows 2 and 3
    (top row x <= 0, bottom row x >= 0), gy >= 0, m of either sign (|s m| vs s m flips
    both).  d/dx likewise with columns 2 | 3.  An inflated or deflated scale (a wrong
    |s m| factor, a dropped corner) fails here, where an upper-bound check would pass."""
    g = _g(1, 6, 7, 2, 3, GEOMS[0], s=s, softmax=softmax)
    Ho, Wo = g.out_hw()
    rs = np.random.RandomState(41)
    shape = (g.N, Ho, Wo, g.G, g.K)
    along = rs.uniform(2.05, 2.95, shape)  # strictly between the split rows/columns
    across = rs.uniform(0.5, 4.5, shape)
    ty, tx = (along, across) if axis == "y" else (across, along)
    dx, dy = _aim_offsets(g, ty, tx)
    m = rs.uniform(0.2, 1.0, shape) * rs.choice([-1.0, 1.0], shape)
    u = rs.uniform(0.1, 1.0, (g.N, g.H, g.W, g.C))
    hh = np.arange(g.H).reshape(1, g.H, 1, 1)
    ww = np.arange(g.W).reshape(1, 1, g.W, 1)
    split = hh if axis == "y" else ww
    x = np.where(split >= 3, u, -u)
    gy = rs.uniform(0.1, 1.0, (g.N, Ho, Wo, g.C))
    om = pack_om(dx, dy, m)
    _, gom, _, goma = oracle.backward(g, x, om, gy, with_abs=True)
    gdx, gdy, _ = unpack_om(gom, g.G, g.K)
    adx, ady, _ = unpack_om(goma, g.G, g.K)
    val, scale = (gdy, ady) if axis == "y" else (gdx, adx)
    assert np.all(scale > 0)
    np.testing.assert_allclose(np.abs(val), scale, rtol=1e-12, atol=0)


def test_softmax_mask_grad_scale_closed_form():
    """DCNv3 mode (R18): dL/dz_k = p_k (gm_k - sum_j p_j gm_j); its scale
    is p_k (|gm|_k + sum_j p_j |gm|_j).  With one tap k0 in the image (the other taps
    pushed far outside, so gm_k = |gm|_k = 0 for them) and x, gy >= 0, the forward gives
    <gy, y> = p_k0 gm_k0 per (pixel, group), hence in closed form:
      k != k0:  scale_k = |grad_k| = p_k <gy, y>,
      k  = k0:  scale = (1 + p_k0) <gy, y>,  |grad| = (1 - p_k0) <gy, y>."""
    g = _g(1, 5, 6, 2, 2, GEOMS[0], softmax=True)
    Ho, Wo = g.out_hw()
    rs = np.random.RandomState(43)
    shape = (g.N, Ho, Wo, g.G, g.K)
    k0 = 4  # centre tap
    dx = rs.uniform(-0.9, 0.9, shape)
    dy = rs.uniform(-0.9, 0.9, shape)
    far = np.arange(g.K) != k0
    dx[..., far] += 100.0
    z = rs.uniform(-2, 2, shape)
    x = rs.uniform(0.1, 1.0, (g.N, g.H, g.W, g.C))
    gy = rs.uniform(0.1, 1.0, (g.N, Ho, Wo, g.C))
    om = pack_om(dx, dy, z)
    y = oracle.forward(g, x, om)
    _, gom, _, goma = oracle.backward(g, x, om, gy, with_abs=True)
    gz, az = unpack_om(gom, g.G, g.K)[2], unpack_om(goma, g.G, g.K)[2]
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    p = e / e.sum(axis=-1, keepdims=True)  # the DCNv3 normalisation over K
    dot = (gy * y).reshape(g.N, Ho, Wo, g.G, g.D).sum(-1)[..., None]
    assert np.all(dot > 0)
    np.testing.assert_allclose(az[..., far], p[..., far] * dot, rtol=1e-12)
    np.testing.assert_allclose(np.abs(gz[..., far]), az[..., far], rtol=1e-12)
    np.testing.assert_allclose(az[..., k0], (1 + p[..., k0]) * dot[..., 0], rtol=1e-12)
    np.testing.assert_allclose(np.abs(gz[..., k0]), (1 - p[..., k0]) * dot[..., 0], rtol=1e-12)
