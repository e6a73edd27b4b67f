"""GPU parity of the full DCNv4 module (R22) through the C ABI:
the tcgen05 GEMMs of csrc/gemm.cu (dcnv4_linear, dcnv4_linear_grad_input,
dcnv4_linear_grad_weight), the fused kernel with a separate value tensor
(dcnv4_module_core_forward) and the whole module forward/backward, against the fp64
oracle (oracle.linear, oracle.module_full_forward / module_full_backward).

Metric: abs-scaled error with the magnitude scale of each product
(|A| |B| summed like the product itself); tolerance 1e-2 for fp16/bf16 (north star).
Each step is checked on the inputs the GPU step actually received, so a rounding flip in
an earlier layer cannot mask or fake an error in a later one; the end-to-end forward is
checked against the oracle chain as well.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2401_06197_b200 as pkg
from paper_2401_06197_b200 import module as mod

pytestmark = pytest.mark.gpu
TDT = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}
TOL = 1e-2


def _rand(shape, dtype, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return ((torch.rand(shape, generator=g) * 2 - 1) * scale).to(TDT[dtype])


def _f(t):
    return t.detach().cpu().double().numpy()


def _err(gpu, ref, scale):
    return oracle.abs_scaled_error(gpu, ref, scale)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("M,K,N,bias", [(1000, 64, 64, True), (4133, 72, 136, False), (257, 512, 320, True),
                                        (128, 128, 512, True), (20000, 64, 200, True)])
def test_linear(dtype, M, K, N, bias):
    dev = torch.device("cuda:0")
    x = _rand((M, K), dtype, 1)
    w = _rand((N, K), dtype, 2, K ** -0.5)
    b = _rand((N,), dtype, 3) if bias else None
    y = mod.linear(x.to(dev), w.to(dev), b.to(dev) if bias else None)
    torch.cuda.synchronize()
    ref = oracle.linear(x, w, b, dtype)
    scale = oracle.linear_abs(np.abs(_f(x)), w, b)
    assert _err(y, ref, scale) <= TOL
    assert np.mean(_f(y) == ref) >= 0.99  # fp32 accumulation, one rounding: nearly all bit-equal


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("M,K,N0,ld0,N1", [(1000, 64, 108, 112, 64), (3000, 128, 216, 216, 128),
                                           (517, 256, 64, 64, 0), (129, 64, 100, 104, 64)])
def test_linear_grad_input_two_segments(dtype, M, K, N0, ld0, N1):
    dev = torch.device("cuda:0")
    gy0 = _rand((M, ld0), dtype, 4)
    gy0[:, N0:] = 0  # padding columns (grad_offset_mask beyond 3GK) are zero
    w0 = _rand((N0, K), dtype, 5, N0 ** -0.5)
    gy1 = _rand((M, N1), dtype, 6) if N1 else None
    w1 = _rand((N1, K), dtype, 7, max(N1, 1) ** -0.5) if N1 else None
    gx = mod.linear_grad_input(gy0.to(dev), w0.to(dev), N0, gy1.to(dev) if N1 else None,
                               w1.to(dev) if N1 else None)
    torch.cuda.synchronize()
    ref = _f(gy0)[:, :N0] @ _f(w0)
    scale = np.abs(_f(gy0)[:, :N0]) @ np.abs(_f(w0))
    if N1:
        ref = ref + _f(gy1) @ _f(w1)
        scale = scale + np.abs(_f(gy1)) @ np.abs(_f(w1))
    assert _err(gx, oracle.round_to(ref, dtype), scale) <= TOL


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("M,K,N,ld", [(1000, 64, 108, 112), (5000, 128, 128, 128), (20000, 64, 64, 64),
                                      (333, 256, 216, 216)])
def test_linear_grad_weight(dtype, M, K, N, ld):
    dev = torch.device("cuda:0")
    x = _rand((M, K), dtype, 8)
    gy = _rand((M, ld), dtype, 9)
    gy[:, N:] = 0
    gw, gb = mod.linear_grad_weight(x.to(dev), gy.to(dev), N)
    torch.cuda.synchronize()
    ref = _f(gy)[:, :N].T @ _f(x)
    scale = np.abs(_f(gy)[:, :N]).T @ np.abs(_f(x))
    assert _err(gw, oracle.round_to(ref, dtype), scale) <= TOL
    rb = _f(gy)[:, :N].sum(0)
    assert _err(gb, oracle.round_to(rb, dtype), np.abs(_f(gy)[:, :N]).sum(0)) <= TOL


def _module_case(N, H, W, G, D, dtype, seed):
    C, J = G * D, 27 * G
    x = _rand((N, H, W, C), dtype, seed)
    rs = np.random.RandomState(seed)
    p = {"w_in": _rand((C, C), dtype, seed + 1, C ** -0.5), "b_in": _rand((C,), dtype, seed + 2, 0.5),
         "w_om": _rand((J, C), dtype, seed + 3, 1.5 * C ** -0.5), "b_om": _rand((J,), dtype, seed + 4, 0.5),
         "w_out": _rand((C, C), dtype, seed + 5, C ** -0.5), "b_out": _rand((C,), dtype, seed + 6, 0.5)}
    del rs
    return x, p


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("N,H,W,G,D", [(1, 16, 16, 4, 16), (2, 19, 13, 8, 16), (1, 14, 14, 4, 32),
                                       (2, 8, 8, 16, 16)])
def test_core_forward_separate_value(dtype, N, H, W, G, D):
    dev = torch.device("cuda:0")
    x, p = _module_case(N, H, W, G, D, dtype, 20)
    v = _rand(x.shape, dtype, 30)
    y = mod.core_forward(x.to(dev), v.to(dev), p["w_om"].to(dev), p["b_om"].to(dev), G)
    torch.cuda.synchronize()
    g = oracle.Geometry(N=N, H=H, W=W, G=G, D=D)
    om = oracle.offset_mask_linear(_f(x).reshape(-1, G * D), p["w_om"], p["b_om"], g.S, dtype)
    ref, ref_abs = oracle.forward(g, v, om.reshape(N, H, W, g.S), with_abs=True)
    assert _err(y, ref, ref_abs) <= TOL


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("N,H,W,G,D", [(2, 16, 16, 4, 16), (1, 21, 11, 8, 16), (1, 14, 14, 4, 32)])
def test_full_module_forward_backward(dtype, N, H, W, G, D):
    dev = torch.device("cuda:0")
    x, p = _module_case(N, H, W, G, D, dtype, 40)
    gy = _rand(x.shape, dtype, 50)
    xd = x.to(dev)
    pd = {k: v.to(dev) for k, v in p.items()}
    y, (v, a) = mod.full_forward(xd, pd, G)
    g = mod.full_backward(xd, pd, G, gy.to(dev), (v, a))
    torch.cuda.synchronize()
    geo = oracle.Geometry(N=N, H=H, W=W, G=G, D=D)
    C, R = G * D, N * H * W
    # end to end against the oracle chain (every layer rounded to T, R22)
    fw = oracle.module_full_forward(geo, x, p, dtype, with_abs=True)
    assert _err(y, fw["y"], fw["y_abs"]) <= TOL
    # step by step on the GPU's own intermediates
    xf, vf, af = _f(x).reshape(R, C), _f(v).reshape(R, C), _f(a).reshape(R, C)
    assert _err(v.reshape(R, C), oracle.linear(xf, p["w_in"], p["b_in"], dtype),
                oracle.linear_abs(np.abs(xf), p["w_in"], p["b_in"])) <= TOL
    Sg = mod.om_stride_for(G)
    om = oracle.offset_mask_linear(xf, p["w_om"], p["b_om"], Sg, dtype).reshape(N, H, W, Sg)
    gs = oracle.Geometry(N=N, H=H, W=W, G=G, D=D, om_stride=Sg)
    a_ref, a_abs = oracle.forward(gs, vf, om, with_abs=True)
    assert _err(a, a_ref, a_abs) <= TOL
    assert _err(y.reshape(R, C), oracle.linear(af, p["w_out"], p["b_out"], dtype),
                oracle.linear_abs(np.abs(af), p["w_out"], p["b_out"])) <= TOL
    gyf = _f(gy).reshape(R, C)
    wo, wi, wm = _f(p["w_out"]), _f(p["w_in"]), _f(p["w_om"])
    assert _err(g["w_out"], oracle.round_to(gyf.T @ af, dtype), np.abs(gyf).T @ np.abs(af)) <= TOL
    assert _err(g["b_out"], oracle.round_to(gyf.sum(0), dtype), np.abs(gyf).sum(0)) <= TOL
    # the DCNv4 backward on the GPU's ga, v, om (recomputed exactly as the oracle's)
    ga = mod.linear_grad_input(gy.to(dev), pd["w_out"])
    torch.cuda.synchronize()
    gaf = _f(ga).reshape(R, C)
    assert _err(gaf, oracle.round_to(gyf @ wo, dtype), np.abs(gyf) @ np.abs(wo)) <= TOL
    gv_ref, gom_ref, gv_abs, gom_abs = oracle.backward(gs, vf, om, gaf, with_abs=True)
    gv, gom = pkg.backward(v, mod.offset_mask_linear(xd, pd["w_om"], pd["b_om"], G, Sg), ga, G)
    torch.cuda.synchronize()
    assert _err(gv, gv_ref, gv_abs) <= TOL
    gvf, gomf = _f(gv).reshape(R, C), _f(gom).reshape(R, Sg)
    J = 27 * G
    assert _err(g["x"].reshape(R, C), oracle.round_to(gomf[:, :J] @ wm + gvf @ wi, dtype),
                np.abs(gomf[:, :J]) @ np.abs(wm) + np.abs(gvf) @ np.abs(wi)) <= TOL
    assert _err(g["w_in"], oracle.round_to(gvf.T @ xf, dtype), np.abs(gvf).T @ np.abs(xf)) <= TOL
    assert _err(g["b_in"], oracle.round_to(gvf.sum(0), dtype), np.abs(gvf).sum(0)) <= TOL
    assert _err(g["w_om"], oracle.round_to(gomf[:, :J].T @ xf, dtype), np.abs(gomf[:, :J]).T @ np.abs(xf)) <= TOL
    assert _err(g["b_om"], oracle.round_to(gomf[:, :J].sum(0), dtype), np.abs(gomf[:, :J]).sum(0)) <= TOL


def test_nn_module_autograd_matches_full_backward():
    dev = torch.device("cuda:0")
    m = pkg.module.DCNv4Module(64, 4, dtype=torch.float16, device=dev)
    with torch.no_grad():
        m.w_om.copy_(_rand(m.w_om.shape, "f16", 60, 0.2).to(dev))
        m.b_om.copy_(_rand(m.b_om.shape, "f16", 61, 0.5).to(dev))
    x = _rand((2, 12, 12, 64), "f16", 62).to(dev).requires_grad_()
    gy = _rand((2, 12, 12, 64), "f16", 63).to(dev)
    m(x).backward(gy)
    params = {k: getattr(m, k).detach() for k in mod.FULL_KEYS}
    y, saved = mod.full_forward(x.detach(), params, 4)
    g = mod.full_backward(x.detach(), params, 4, gy, saved)
    torch.cuda.synchronize()
    # grad_input of the DCNv4 step and the grad_weight splits sum with fp32 atomics: equal
    # up to rounding order, not bit for bit
    def close(a, b):
        a, b = a.float(), b.float()
        return bool(((a - b).abs() <= 2e-2 * b.abs().max().clamp_min(1e-6)).all())
    assert close(x.grad, g["x"])
    for k in mod.FULL_KEYS:
        assert torch.isfinite(getattr(m, k).grad.float()).all()
        assert close(getattr(m, k).grad, g[k]), k


# ---------------------------------------------------------------- fp32: 3xTF32 GEMMs
@pytest.mark.parametrize("M,K,N", [(1000, 64, 64), (4133, 72, 136), (257, 512, 320)])
def test_linear_f32_3xtf32(M, K, N):
    """fp32 linear on the tf32 tensor cores as 3xTF32 meets the fp32 bar (1e-5)."""
    dev = torch.device("cuda:0")
    x = _rand((M, K), "f32", 11)
    w = _rand((N, K), "f32", 12, K ** -0.5)
    b = _rand((N,), "f32", 13)
    y = mod.linear(x.to(dev), w.to(dev), b.to(dev))
    torch.cuda.synchronize()
    ref = oracle.linear(x, w, b)
    assert _err(y, ref, oracle.linear_abs(np.abs(_f(x)), w, b)) <= 1e-5


def test_linear_grads_f32_3xtf32():
    dev = torch.device("cuda:0")
    M, K, N0, N1 = 3000, 64, 108, 64
    gy0, w0 = _rand((M, N0), "f32", 14), _rand((N0, K), "f32", 15, N0 ** -0.5)
    gy1, w1 = _rand((M, N1), "f32", 16), _rand((N1, K), "f32", 17, N1 ** -0.5)
    gx = mod.linear_grad_input(gy0.to(dev), w0.to(dev), N0, gy1.to(dev), w1.to(dev))
    x = _rand((M, K), "f32", 18)
    gw, gb = mod.linear_grad_weight(x.to(dev), gy0.to(dev), N0)
    torch.cuda.synchronize()
    ref = _f(gy0) @ _f(w0) + _f(gy1) @ _f(w1)
    assert _err(gx, ref, np.abs(_f(gy0)) @ np.abs(_f(w0)) + np.abs(_f(gy1)) @ np.abs(_f(w1))) <= 1e-5
    assert _err(gw, _f(gy0).T @ _f(x), np.abs(_f(gy0)).T @ np.abs(_f(x))) <= 1e-5
    assert _err(gb, _f(gy0).sum(0), np.abs(_f(gy0)).sum(0)) <= 1e-5


def test_full_module_f32():
    dev = torch.device("cuda:0")
    N, H, W, G, D = 2, 12, 12, 4, 16
    x, p = _module_case(N, H, W, G, D, "f32", 70)
    gy = _rand(x.shape, "f32", 71)
    xd, pd = x.to(dev), {k: v.to(dev) for k, v in p.items()}
    y, saved = mod.full_forward(xd, pd, G)
    g = mod.full_backward(xd, pd, G, gy.to(dev), saved)
    torch.cuda.synchronize()
    geo = oracle.Geometry(N=N, H=H, W=W, G=G, D=D)
    fw = oracle.module_full_forward(geo, x, p, "f32", with_abs=True)
    assert _err(y, fw["y"], fw["y_abs"]) <= 1e-5
    bw = oracle.module_full_backward(geo, x, p, gy, "f32")
    R, C = N * H * W, G * D
    # scales: |terms| summed like each product (chained magnitudes of the inputs)
    xf, gyf = np.abs(_f(x).reshape(R, C)), np.abs(_f(gy).reshape(R, C))
    assert np.abs(_f(g["w_out"]) - bw["w_out"]).max() <= 1e-5 * (gyf.T @ np.abs(fw["a"].reshape(R, C))).max()
    assert np.abs(_f(g["x"]) - bw["x"]).max() <= 1e-4 * np.abs(bw["x"]).max()


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("dtype", ["f16", "bf16", "f32"])
@pytest.mark.parametrize("M,K,N", [(1, 16, 8), (127, 24, 72), (129, 64, 8), (300, 8, 264)])
def test_linear_edge_shapes(dtype, M, K, N):
    """Single row, fewer rows than one 128-row tile, K below one k block, ragged N."""
    if dtype == "f32":
        K, N = max(4, K), max(4, N)
    dev = torch.device("cuda:0")
    x = _rand((M, K), dtype, 80)
    w = _rand((N, K), dtype, 81, K ** -0.5)
    b = _rand((N,), dtype, 82)
    y = mod.linear(x.to(dev), w.to(dev), b.to(dev))
    torch.cuda.synchronize()
    ref = oracle.linear(x, w, b, dtype if dtype != "f32" else "f64")
    tol = 1e-5 if dtype == "f32" else TOL
    assert _err(y, ref, oracle.linear_abs(np.abs(_f(x)), w, b)) <= tol


@pytest.mark.parametrize("dtype", ["f16", "f32"])
@pytest.mark.parametrize("M", [1, 37, 130])
def test_linear_grad_weight_few_rows(dtype, M):
    """The split-K grad_weight with fewer rows than one k block (zero-filled tail)."""
    dev = torch.device("cuda:0")
    K, N = 64, 24
    x = _rand((M, K), dtype, 83)
    gy = _rand((M, N), dtype, 84)
    gw, gb = mod.linear_grad_weight(x.to(dev), gy.to(dev))
    torch.cuda.synchronize()
    ref = _f(gy).T @ _f(x)
    tol = 1e-5 if dtype == "f32" else TOL
    assert _err(gw, ref, np.abs(_f(gy)).T @ np.abs(_f(x))) <= tol
    assert _err(gb, _f(gy).sum(0), np.abs(_f(gy)).sum(0)) <= tol


def test_full_module_softmax_bf16():
    """DCNv3 mode (softmax over K, R18) through the full module, bf16."""
    dev = torch.device("cuda:0")
    N, H, W, G, D = 1, 14, 10, 4, 16
    x, p = _module_case(N, H, W, G, D, "bf16", 90)
    xd, pd = x.to(dev), {k: v.to(dev) for k, v in p.items()}
    y, saved = mod.full_forward(xd, pd, G, softmax=True)
    gy = _rand(x.shape, "bf16", 91)
    g = mod.full_backward(xd, pd, G, gy.to(dev), saved, softmax=True)
    torch.cuda.synchronize()
    geo = oracle.Geometry(N=N, H=H, W=W, G=G, D=D, softmax=True)
    fw = oracle.module_full_forward(geo, x, p, "bf16", with_abs=True)
    assert _err(y, fw["y"], fw["y_abs"]) <= TOL
    for k in mod.FULL_KEYS:
        assert torch.isfinite(g[k].float()).all()
