"""Pins of the full-module oracle (R22), CPU only.

oracle.module_full_forward / module_full_backward are the full DCNv4 module of P:198 /
P:1006-1009: v = linear(x; W_in), om = linear(x; W_om), a = DCNv4(v, om),
y = linear(a; W_out), and its backward.  What fixes the expected values:
  * torch autograd through an independent fp64 torch model of the module (F.linear +
    the grid_sample formulation of Eq. (1) from test_oracle_pins) for y and every
    gradient (x, W_in, b_in, W_om, b_om, W_out, b_out);
  * the 1x1 projections against torch conv2d with a 1x1 kernel;
  * identity projections reduce the full module to the lightweight one exactly.
A transposed weight, a dropped bias gradient, gx missing one of its two paths, or the
offsets read from v instead of x fails one of them.
"""
import numpy as np
import torch
import torch.nn.functional as F

import oracle
from tests.helpers import geom
from tests.test_oracle_pins import _grid_sample_model


def _params(C, G, K, seed, dtype_round=None):
    rs = np.random.RandomState(seed)
    J = 3 * G * K
    p = {"w_in": rs.uniform(-1, 1, (C, C)) / np.sqrt(C), "b_in": rs.uniform(-0.5, 0.5, C),
         "w_om": rs.uniform(-1, 1, (J, C)) / np.sqrt(C), "b_om": rs.uniform(-0.5, 0.5, J),
         "w_out": rs.uniform(-1, 1, (C, C)) / np.sqrt(C), "b_out": rs.uniform(-0.5, 0.5, C)}
    return p


def _torch_module(g, x, p):
    """Independent fp64 torch model: F.linear for the three linears, grid_sample for
    Eq. (1) (offsets / masks unpacked from the om channels, layout R3)."""
    N, H, W, C = x.shape
    v = F.linear(x, p["w_in"], p["b_in"])
    om = F.linear(x, p["w_om"], p["b_om"])
    K = g.K
    omg = om.reshape(N, H, W, g.G, 3 * K)
    dx, dy, m = omg[..., 0:2 * K:2], omg[..., 1:2 * K:2], omg[..., 2 * K:]
    a = _grid_sample_model(g, v, dx, dy, m)
    return F.linear(a, p["w_out"], p["b_out"])


def test_full_module_matches_torch_autograd():
    g = geom(N=2, H=6, W=7, G=2, D=4)
    rs = np.random.RandomState(5)
    x = rs.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    p = _params(g.C, g.G, g.K, 6)
    gy = rs.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    fw = oracle.module_full_forward(g, x, p)
    bw = oracle.module_full_backward(g, x, p, gy)
    xt = torch.tensor(x, requires_grad=True)
    pt = {k: torch.tensor(v, requires_grad=True) for k, v in p.items()}
    yt = _torch_module(g, xt, pt)
    (yt * torch.from_numpy(gy)).sum().backward()
    np.testing.assert_allclose(fw["y"], yt.detach().numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(bw["x"], xt.grad.numpy(), rtol=0, atol=1e-10)
    for k in p:
        np.testing.assert_allclose(bw[k], pt[k].grad.numpy(), rtol=0, atol=1e-10, err_msg=k)


def test_projections_are_1x1_convolutions():
    rs = np.random.RandomState(8)
    x = rs.uniform(-1, 1, (2, 5, 6, 12))
    w = rs.uniform(-1, 1, (20, 12))
    b = rs.uniform(-1, 1, 20)
    y = oracle.linear(x.reshape(-1, 12), w, b).reshape(2, 5, 6, 20)
    ref = F.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2), torch.from_numpy(w)[:, :, None, None],
                   torch.from_numpy(b)).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-13)


def test_identity_projections_give_the_lightweight_module():
    g = geom(N=1, H=8, W=5, G=2, D=8)
    rs = np.random.RandomState(9)
    x = oracle.round_to(rs.uniform(-1, 1, (g.N, g.H, g.W, g.C)), "f16")
    p = _params(g.C, g.G, g.K, 10)
    p.update(w_in=np.eye(g.C), b_in=np.zeros(g.C), w_out=np.eye(g.C), b_out=np.zeros(g.C))
    p["w_om"] = oracle.round_to(p["w_om"], "f16")
    p["b_om"] = oracle.round_to(p["b_om"], "f16")
    full = oracle.module_full_forward(g, x, p, "f16")
    light = oracle.round_to(oracle.module_forward(g, x, p["w_om"], p["b_om"], "f16"), "f16")
    np.testing.assert_array_equal(full["y"], light)


def test_offsets_come_from_the_input_not_the_value():
    """R22: with W_in = 2 I the samples double but the offsets do not move: y = 2 y(W_in = I)."""
    g = geom(N=1, H=6, W=6, G=1, D=8)
    rs = np.random.RandomState(11)
    x = rs.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    p = _params(g.C, g.G, g.K, 12)
    p.update(w_in=np.eye(g.C), b_in=np.zeros(g.C), w_out=np.eye(g.C), b_out=np.zeros(g.C))
    y1 = oracle.module_full_forward(g, x, p)["y"]
    p["w_in"] = 2 * np.eye(g.C)
    y2 = oracle.module_full_forward(g, x, p)["y"]
    np.testing.assert_allclose(y2, 2 * y1, rtol=0, atol=1e-13)


def test_abs_scale_bounds_the_output():
    g = geom(N=1, H=5, W=6, G=2, D=4)
    rs = np.random.RandomState(13)
    x = rs.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    p = _params(g.C, g.G, g.K, 14)
    fw = oracle.module_full_forward(g, x, p, with_abs=True)
    assert np.all(np.abs(fw["y"]) <= fw["y_abs"] + 1e-12)
    # non-negative data: the scale is the value (x, W, b >= 0 and m >= 0)
    pa = {k: np.abs(v) for k, v in p.items()}
    fa = oracle.module_full_forward(g, np.abs(x), pa, with_abs=True)
    np.testing.assert_allclose(fa["y"], fa["y_abs"], rtol=1e-12)
