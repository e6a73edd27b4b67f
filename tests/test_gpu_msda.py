"""GPU parity of multi-scale deformable attention (NEXT-3, include/msda.h) against the fp64
oracle (oracle/msda_oracle.c), element by element with the abs-scaled error metric of
SURVEY 8(c).4: fp32 max e <= 1e-5, fp16/bf16 <= 1e-2.  grad_loc entries whose fp64 pixel
coordinate lies within 1e-5 of an integer (a kink: several sub-gradients are valid) are
masked and counted.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2401_06197_b200 as pkg
from paper_2401_06197_b200 import msda
from tests.test_gpu_parity import QFLOOR, TDT, TOL, _err

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def _kink_mask(g, loc64, eps=1e-5):
    mask = np.zeros(loc64.shape, bool)
    for l, (H, W) in enumerate(g.shapes):
        px = loc64[:, :, :, l, :, 0] * W - 0.5
        py = loc64[:, :, :, l, :, 1] * H - 0.5
        mask[:, :, :, l, :, 0] = np.abs(px - np.round(px)) < eps
        mask[:, :, :, l, :, 1] = np.abs(py - np.round(py)) < eps
    return mask


def run_msda(g, dtype="f32", loc_range=(-0.1, 1.1), backward=True, check_images=None,
             inputs=None):
    if inputs is None:
        value, loc, attn, gout = synth.make_msda_case(g.N, g.Lq, g.M, g.D, g.P, g.shapes, dtype,
                                                      loc_range=loc_range)
    else:
        value, loc, attn, gout = inputs
    vd, ld, ad, gd = (t.to(DEV) for t in (value, loc, attn, gout))
    out = msda.forward(vd, ld, ad, g.shapes)
    if backward:
        gv, gl, ga = msda.backward(vd, ld, ad, gd, g.shapes)
    torch.cuda.synchronize()
    sel = list(range(g.N)) if check_images is None else list(check_images)
    gs = oracle.MSDAGeometry(**{**g.__dict__, "N": len(sel)})
    vs, ls, as_, gos = value[sel], loc[sel], attn[sel], gout[sel]
    qf = QFLOOR[dtype]
    ref, ref_abs = oracle.msda_forward(gs, vs, ls, as_, with_abs=True)
    errs = {"out": _err(out[sel], ref, ref_abs, qfloor=qf)}
    if backward:
        rgv, rgl, rga, agv, agl, aga = oracle.msda_backward(gs, vs, ls, as_, gos, with_abs=True)
        mask = _kink_mask(gs, ls.double().numpy())
        errs["grad_value"] = _err(gv[sel], rgv, agv, qfloor=qf)
        errs["grad_loc"] = _err(gl[sel], rgl, agl, mask, qfloor=qf)
        errs["grad_attn"] = _err(ga[sel], rga, aga, qfloor=qf)
        errs["masked"] = int(mask.sum())
    return errs


def _ok(errs, dtype):
    tol = TOL[dtype]
    bad = {k: v for k, v in errs.items() if k != "masked" and not (v <= tol)}
    assert not bad, f"{dtype}: {errs}"


def G(N, Lq, M, D, P, shapes):
    return oracle.MSDAGeometry(N=N, Lq=Lq, M=M, D=D, P=P, shapes=tuple(shapes))


CASES = [
    ("detr_small", G(2, 37, 8, 32, 4, [(12, 17), (6, 9), (3, 5), (2, 3)])),
    ("one_level", G(1, 20, 2, 32, 1, [(9, 11)])),
    ("ragged_heads", G(3, 11, 3, 16, 3, [(7, 5), (4, 3)])),
    ("D64_P8", G(1, 9, 4, 64, 8, [(6, 6), (3, 3), (2, 2)])),
    ("D8", G(2, 13, 5, 8, 2, [(5, 9), (3, 4), (1, 1)])),
    ("eight_levels", G(1, 6, 2, 32, 2, [(9, 9), (7, 8), (5, 6), (4, 4), (3, 3), (2, 2), (1, 2), (1, 1)])),
    ("tiny_levels", G(2, 7, 1, 16, 5, [(1, 1), (1, 2), (2, 1)])),
]


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("name,g", CASES, ids=[c[0] for c in CASES])
def test_msda_parity(name, g, dtype):
    _ok(run_msda(g, dtype), dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_msda_all_outside_and_far(dtype):
    g = G(2, 9, 2, 32, 2, [(6, 7), (3, 4)])
    _ok(run_msda(g, dtype, loc_range=(-3.0, 4.0)), dtype)
    value, loc, attn, gout = synth.make_msda_case(1, 5, 2, 32, 2, g.shapes, dtype, loc_range=(1.5, 2.0))
    vd, ld, ad, gd = (t.to(DEV) for t in (value, loc, attn, gout))
    out = msda.forward(vd, ld, ad, g.shapes)
    gv, gl, ga = msda.backward(vd, ld, ad, gd, g.shapes)
    assert not out.any() and not gv.any() and not gl.any() and not ga.any()


def test_msda_pixel_centres_exact():
    shapes = ((5, 7), (3, 4))
    g = G(1, 4, 2, 16, 1, shapes)
    value, _, attn, _ = synth.make_msda_case(1, 4, 2, 16, 1, shapes, "f32")
    loc = torch.empty((1, 4, 2, 2, 1, 2))
    rng = np.random.default_rng(3)
    for l, (H, W) in enumerate(shapes):
        loc[..., l, :, 0] = torch.from_numpy((rng.integers(0, W, (1, 4, 2, 1)) + 0.5) / W).float()
        loc[..., l, :, 1] = torch.from_numpy((rng.integers(0, H, (1, 4, 2, 1)) + 0.5) / H).float()
    out = msda.forward(value.to(DEV), loc.to(DEV), attn.to(DEV), shapes).cpu().double().numpy()
    ref = oracle.msda_forward(g, value, loc, attn)
    assert np.abs(out - ref).max() <= 1e-6 * np.abs(ref).max()


def test_msda_empty_and_zero_queries():
    shapes = ((4, 4),)
    v = torch.randn(0, 16, 2, 32, device=DEV)
    out = msda.forward(v, torch.zeros(0, 3, 2, 1, 2, 2, device=DEV), torch.zeros(0, 3, 2, 1, 2, device=DEV), shapes)
    assert out.shape == (0, 3, 2, 32)
    v = torch.randn(2, 16, 2, 32, device=DEV)
    lo = torch.zeros(2, 0, 2, 1, 2, 2, device=DEV)
    at = torch.zeros(2, 0, 2, 1, 2, device=DEV)
    gv, gl, ga = msda.backward(v, lo, at, torch.zeros(2, 0, 2, 32, device=DEV), shapes,
                               grad_value=torch.full_like(v, 7.0))
    assert not gv.any()


def test_msda_deterministic_forward_and_autograd():
    g = CASES[0][1]
    value, loc, attn, gout = (t.to(DEV) for t in synth.make_msda_case(
        g.N, g.Lq, g.M, g.D, g.P, g.shapes, "f32"))
    a = msda.forward(value, loc, attn, g.shapes)
    b = msda.forward(value, loc, attn, g.shapes)
    assert torch.equal(a, b)
    v, lc, at = (t.clone().requires_grad_() for t in (value, loc, attn))
    msda.msda(v, lc, at, g.shapes).backward(gout)
    gv, gl, ga = msda.backward(value, loc, attn, gout, g.shapes)
    assert torch.equal(lc.grad, gl) and torch.equal(at.grad, ga)
    assert (v.grad - gv).abs().max().item() <= 1e-6 * gv.abs().max().item()


def test_msda_randomized_configs():
    rng = np.random.default_rng(20240111)
    for _ in range(25):
        L = int(rng.integers(1, 5))
        shapes = [(int(rng.integers(1, 14)), int(rng.integers(1, 14))) for _ in range(L)]
        dtype = ["f32", "f16", "bf16"][int(rng.integers(0, 3))]
        D = int(rng.choice([8, 16, 32, 64] if dtype != "f32" else [4, 8, 16, 32, 64]))
        g = G(int(rng.integers(1, 3)), int(rng.integers(1, 30)), int(rng.integers(1, 9)), D,
              int(rng.integers(1, 6)), shapes)
        errs = run_msda(g, dtype)
        tol = TOL[dtype]
        assert all(v <= tol for k, v in errs.items() if k != "masked"), (g, dtype, errs)


# Deformable-DETR encoder shapes (bench workload "msda"): sampled images at full size
DETR = G(2, 0, 8, 32, 4, [(100, 150), (50, 75), (25, 38), (13, 19)])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_msda_full_size_encoder(dtype):
    S = sum(h * w for h, w in DETR.shapes)
    g = oracle.MSDAGeometry(N=2, Lq=S, M=8, D=32, P=4, shapes=DETR.shapes)
    _ok(run_msda(g, dtype, check_images=[1]), dtype)
