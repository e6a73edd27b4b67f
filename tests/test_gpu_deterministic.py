"""Deterministic backward (R19): grad_input accumulated as
per-image int64 fixed point.  Checked against the fp64 oracle with the same tolerances as
the default path, and for bit-reproducibility across repeated runs, CTA grids (persistent
vs one CTA per tile) and batch splits.
"""
import os

import pytest
import torch

import synth
import paper_2401_06197_b200 as pkg
from tests.test_gpu_parity import CASES, TDT, _assert_tol, _geom, run_case

pytestmark = pytest.mark.gpu

DET_CASES = [c for c in CASES if c[0] in (
    "c1_tiny", "ragged", "stride2_pad0", "k5x5", "scale0.5", "om_stride_pad", "zero_offsets_kinks",
    "u8_offsets", "D64", "G80_wide", "softmax_v3", "halo_G4_u8", "halo_G8_ragged",
    "halo_G4_softmax")]


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("name,g,offsets", DET_CASES, ids=[c[0] for c in DET_CASES])
def test_deterministic_parity(name, g, offsets, dtype):
    _assert_tol(run_case(g, dtype, offsets, deterministic=True), dtype)


def _inputs(N, H, W, G, dtype, offsets="u2", images=None):
    x, om, gy = synth.make_case(N, H, W, G, 16, H, W, 9, 27 * G, dtype, images=images,
                                offsets=offsets)
    dev = torch.device("cuda:0")
    return x.to(dev), om.to(dev), gy.to(dev)


def _det_backward_with_switch(env: dict, N, H, W, G, dtype, offsets, reps=1):
    """grad_input of `reps` deterministic backward calls in a fresh process whose
    environment holds an ablation switch (the library reads its switches once, at first
    use: csrc/ablation.h), on the same seeded inputs as _inputs()."""
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "gx.pt")
        code = ("import torch, sys; sys.path.insert(0, %r)\n"
                "from tests.test_gpu_deterministic import _inputs\n"
                "import paper_2401_06197_b200 as pkg\n"
                "x, om, gy = _inputs(%d, %d, %d, %d, %r, %r)\n"
                "r = [pkg.backward(x, om, gy, group=%d, deterministic=True)[0].cpu() for _ in range(%d)]\n"
                "torch.save(r, %r)\n") % (root, N, H, W, G, dtype, offsets, G, reps, out)
        subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env),
                       check=True, timeout=300)
        return torch.load(out)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("offsets", ["u2", "u8"])
def test_bit_identical_runs_grids_and_splits(dtype, offsets):
    N, H, W, G = 6, 28, 28, 8
    x, om, gy = _inputs(N, H, W, G, dtype, offsets)
    ref, gom_ref = pkg.backward(x, om, gy, group=G, deterministic=True)
    for _ in range(3):
        gx, gom = pkg.backward(x, om, gy, group=G, deterministic=True)
        assert torch.equal(gx, ref) and torch.equal(gom, gom_ref)
    # a different CTA -> tile assignment (one CTA per tile instead of a persistent grid)
    (gx,) = _det_backward_with_switch({"DCNV4_NONPERSISTENT": "1"}, N, H, W, G, dtype, offsets)
    assert torch.equal(gx, ref.cpu())
    # the global-gather kernel agrees with the TMA-halo kernel only within tolerance, but
    # is itself reproducible
    a, b = _det_backward_with_switch({"DCNV4_BWD_PATH": "g"}, N, H, W, G, dtype, offsets, reps=2)
    assert torch.equal(a, b)
    # batch split: per-image scale, so a sub-batch reproduces its slice bit for bit
    for lo, hi in ((0, 1), (2, 5), (5, 6)):
        part, _ = pkg.backward(x[lo:hi].contiguous(), om[lo:hi].contiguous(),
                               gy[lo:hi].contiguous(), group=G, deterministic=True)
        assert torch.equal(part, ref[lo:hi])


def test_default_path_close_to_deterministic():
    x, om, gy = _inputs(4, 56, 56, 4, "f32")
    a, _ = pkg.backward(x, om, gy, group=4)
    b, _ = pkg.backward(x, om, gy, group=4, deterministic=True)
    scale = a.abs().max().item()
    assert (a - b).abs().max().item() <= 1e-5 * scale


def test_out_of_range_image_is_nan_others_unaffected():
    N, H, W, G = 3, 14, 14, 4
    x, om, gy = _inputs(N, H, W, G, "f32")
    ref, _ = pkg.backward(x, om, gy, group=G, deterministic=True)
    gy2 = gy.clone()
    gy2[1] *= 2.0 ** 70  # max|gy| of image 1 outside [2^-64, 2^64)
    gx, _ = pkg.backward(x, om, gy2, group=G, deterministic=True)
    assert torch.isnan(gx[1]).all()
    assert torch.equal(gx[0], ref[0]) and torch.equal(gx[2], ref[2])
    gy3 = gy.clone()
    gy3[2, 3, 4, 5] = float("nan")
    gx, _ = pkg.backward(x, om, gy3, group=G, deterministic=True)
    assert torch.isnan(gx[2]).all() and torch.equal(gx[0], ref[0])


def test_zero_grad_output_gives_exact_zero():
    x, om, gy = _inputs(2, 10, 10, 2, "f16")
    gx, _ = pkg.backward(x, om, torch.zeros_like(gy), group=2, deterministic=True)
    assert not gx.any()


def test_workspace_size_and_autograd_flag():
    p = pkg.make_params(2, 10, 10, 2, 16, deterministic=True)
    assert pkg.workspace_bytes(p, torch.float32) == 2 * 10 * 10 * 32 * 8 + 16
    assert pkg.workspace_bytes(pkg.make_params(2, 10, 10, 2, 16), torch.float32) == 0
    x, om, gy = _inputs(2, 10, 10, 2, "f32")
    xa, oma = x.clone().requires_grad_(), om.clone().requires_grad_()
    pkg.dcnv4(xa, oma, group=2, deterministic=True).backward(gy)
    gx, gom = pkg.backward(x, om, gy, group=2, deterministic=True)
    assert torch.equal(xa.grad, gx) and torch.equal(oma.grad, gom)
