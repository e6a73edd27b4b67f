"""Pins of the multi-scale deformable attention oracle (NEXT-3, R20) against
things other than itself: torch grid_sample (align_corners=False, zero padding) per
level with autograd for every gradient, closed forms (constant value, pixel centres,
affine ramp, all samples outside), linearity and the adjoint identity.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

SHAPES = [((5, 7),), ((6, 5), (3, 3)), ((8, 9), (4, 5), (2, 3), (1, 2))]


def _grid_sample_ref(g, value, loc, attn):
    """out via torch grid_sample in fp64 (differentiable in all three inputs)."""
    outs = []
    start = 0
    N = value.shape[0]
    res = torch.zeros((N, g.Lq, g.M, g.D), dtype=torch.float64)
    for l, (H, W) in enumerate(g.shapes):
        v = value[:, start:start + H * W]                        # [N, HW, M, D]
        v = v.reshape(N, H, W, g.M, g.D).permute(0, 3, 4, 1, 2)  # [N, M, D, H, W]
        v = v.reshape(N * g.M, g.D, H, W)
        grid = loc[:, :, :, l] * 2.0 - 1.0                       # [N, Lq, M, P, 2] (x, y)
        grid = grid.permute(0, 2, 1, 3, 4).reshape(N * g.M, g.Lq, g.P, 2)
        smp = F.grid_sample(v, grid, mode="bilinear", padding_mode="zeros",
                            align_corners=False)                 # [N*M, D, Lq, P]
        smp = smp.reshape(N, g.M, g.D, g.Lq, g.P)
        a = attn[:, :, :, l].permute(0, 2, 1, 3)                 # [N, M, Lq, P]
        res = res + torch.einsum("nmdqp,nmqp->nqmd", smp, a)
        start += H * W
        outs.append(smp)
    return res


def _case(shapes, N=2, Lq=5, M=3, D=4, P=3, loc_range=(-0.1, 1.1)):
    g = oracle.MSDAGeometry(N=N, Lq=Lq, M=M, D=D, P=P, shapes=tuple(shapes))
    value, loc, attn, gout = synth.make_msda_case(N, Lq, M, D, P, shapes, "f32",
                                                  loc_range=loc_range)
    return g, value.double(), loc.double(), attn.double(), gout.double()


@pytest.mark.parametrize("shapes", SHAPES, ids=["L1", "L2", "L4"])
def test_forward_matches_grid_sample(shapes):
    g, value, loc, attn, _ = _case(shapes)
    ref = _grid_sample_ref(g, value, loc, attn).numpy()
    out = oracle.msda_forward(g, value, loc, attn)
    assert np.abs(out - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("shapes", SHAPES, ids=["L1", "L2", "L4"])
def test_backward_matches_grid_sample_autograd(shapes):
    g, value, loc, attn, gout = _case(shapes)
    v, lc, a = (t.clone().requires_grad_() for t in (value, loc, attn))
    _grid_sample_ref(g, v, lc, a).backward(gout)
    gval, gloc, gattn = oracle.msda_backward(g, value, loc, attn, gout)
    for got, want in ((gval, v.grad), (gloc, lc.grad), (gattn, a.grad)):
        want = want.numpy()
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_constant_value_partition_of_unity():
    # all samples strictly inside the pixel-centre hull: pixel coords in [0, H-1] x [0, W-1]
    shapes = ((6, 7), (3, 4))
    g = oracle.MSDAGeometry(N=1, Lq=4, M=2, D=3, P=2, shapes=shapes)
    rng = np.random.default_rng(0)
    loc = np.empty((1, 4, 2, 2, 2, 2))
    for l, (H, W) in enumerate(shapes):
        loc[:, :, :, l, :, 0] = (rng.uniform(0, W - 1, (1, 4, 2, 2)) + 0.5) / W
        loc[:, :, :, l, :, 1] = (rng.uniform(0, H - 1, (1, 4, 2, 2)) + 0.5) / H
    attn = rng.uniform(-1, 1, (1, 4, 2, 2, 2))
    value = np.full((1, g.S, 2, 3), 2.5)
    out = oracle.msda_forward(g, value, loc, attn)
    np.testing.assert_allclose(out, 2.5 * attn.sum(axis=(3, 4))[..., None].repeat(3, -1), rtol=0,
                               atol=1e-13)
    _, gloc, _ = oracle.msda_backward(g, value, loc, attn, np.ones((1, 4, 2, 3)))
    assert np.abs(gloc).max() <= 1e-12


def test_pixel_centres_are_exact():
    shapes = ((4, 5),)
    g = oracle.MSDAGeometry(N=1, Lq=1, M=1, D=2, P=1, shapes=shapes)
    value = np.arange(4 * 5 * 2, dtype=np.float64).reshape(1, 20, 1, 2)
    for (h, w) in [(0, 0), (3, 4), (2, 1)]:
        loc = np.array([(w + 0.5) / 5, (h + 0.5) / 4]).reshape(1, 1, 1, 1, 1, 2)
        out = oracle.msda_forward(g, value, loc, np.ones((1, 1, 1, 1, 1)))
        np.testing.assert_array_equal(out[0, 0, 0], value[0, h * 5 + w, 0])


def test_affine_ramp_closed_form():
    # V(h, w, c) = alpha*h + beta*w + gamma_c is reproduced exactly by bilinear sampling, so
    # out = sum a*(alpha*h + beta*w + gamma_c) and d out/d x = a * W * beta (no kinks)
    shapes = ((7, 9), (4, 6))
    alpha, beta = 0.75, -1.25
    gamma = np.array([0.5, -2.0, 3.0])
    g = oracle.MSDAGeometry(N=1, Lq=3, M=2, D=3, P=2, shapes=shapes)
    vals = []
    for (H, W) in shapes:
        hh, ww = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        v = alpha * hh[..., None] + beta * ww[..., None] + gamma
        vals.append(np.repeat(v.reshape(H * W, 1, 3), 2, axis=1))
    value = np.concatenate(vals)[None]
    rng = np.random.default_rng(1)
    loc = np.empty((1, 3, 2, 2, 2, 2))
    pix = np.empty((1, 3, 2, 2, 2, 2))
    for l, (H, W) in enumerate(shapes):
        pw = rng.uniform(0, W - 1, (1, 3, 2, 2))
        ph = rng.uniform(0, H - 1, (1, 3, 2, 2))
        loc[:, :, :, l, :, 0] = (pw + 0.5) / W
        loc[:, :, :, l, :, 1] = (ph + 0.5) / H
        pix[:, :, :, l, :, 0], pix[:, :, :, l, :, 1] = pw, ph
    attn = rng.uniform(-1, 1, (1, 3, 2, 2, 2))
    want = np.einsum("nqmlp,nqmlpc->nqmc", attn,
                     alpha * pix[..., 1:2] + beta * pix[..., 0:1] + gamma)
    out = oracle.msda_forward(g, value, loc, attn)
    np.testing.assert_allclose(out, want, rtol=0, atol=1e-12)
    gout = rng.uniform(-1, 1, (1, 3, 2, 3))
    _, gloc, gattn = oracle.msda_backward(g, value, loc, attn, gout)
    sg = gout.sum(-1)[:, :, :, None, None]
    Ws = np.array([w for _, w in shapes])[None, None, None, :, None]
    Hs = np.array([h for h, _ in shapes])[None, None, None, :, None]
    np.testing.assert_allclose(gloc[..., 0], attn * Ws * beta * sg, rtol=0, atol=1e-11)
    np.testing.assert_allclose(gloc[..., 1], attn * Hs * alpha * sg, rtol=0, atol=1e-11)
    want_ga = np.einsum("nqmc,nqmlpc->nqmlp", gout,
                        alpha * pix[..., 1:2] + beta * pix[..., 0:1] + gamma)
    np.testing.assert_allclose(gattn, want_ga, rtol=0, atol=1e-11)


def test_samples_outside_give_zero():
    g, value, loc, attn, gout = _case(SHAPES[1], loc_range=(1.5, 3.0))
    out = oracle.msda_forward(g, value, loc, attn)
    gval, gloc, gattn = oracle.msda_backward(g, value, loc, attn, gout)
    assert not out.any() and not gval.any() and not gloc.any() and not gattn.any()


def test_linearity_and_adjoint():
    g, value, loc, attn, gout = _case(SHAPES[2])
    v2 = torch.rand_like(value)
    o1 = oracle.msda_forward(g, value, loc, attn)
    o2 = oracle.msda_forward(g, v2, loc, attn)
    o12 = oracle.msda_forward(g, 2.0 * value - 3.0 * v2, loc, attn)
    np.testing.assert_allclose(o12, 2.0 * o1 - 3.0 * o2, rtol=0, atol=1e-12)
    a2 = torch.rand_like(attn)
    np.testing.assert_allclose(oracle.msda_forward(g, value, loc, attn + a2),
                               o1 + oracle.msda_forward(g, value, loc, a2), rtol=0, atol=1e-12)
    gval, _, _ = oracle.msda_backward(g, value, loc, attn, gout)
    lhs = float((gout.numpy() * o1).sum())
    rhs = float((gval * value.numpy()).sum())
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
    # Euler: <gattn, attn> = <gout, out> (out is linear in attn)
    _, _, gattn = oracle.msda_backward(g, value, loc, attn, gout)
    assert abs(float((gattn * attn.numpy()).sum()) - lhs) <= 1e-12 * max(1.0, abs(lhs))


def test_abs_pass_bounds_values():
    g, value, loc, attn, gout = _case(SHAPES[1])
    out, oa = oracle.msda_forward(g, value, loc, attn, with_abs=True)
    assert (np.abs(out) <= oa + 1e-15).all()
    gval, gloc, gattn, gva, gla, gaa = oracle.msda_backward(g, value, loc, attn, gout, with_abs=True)
    for x, a in ((gval, gva), (gloc, gla), (gattn, gaa)):
        assert (np.abs(x) <= a + 1e-15).all()
