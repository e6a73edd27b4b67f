"""The host-streaming pipeline (paper_2401_06197_b200/pipeline.py) is plumbing only: a
chunked three-stream pass over a host batch must give the same outputs as one direct
call per tensor (forward and grad_offset_mask bit-identical: they are bit-deterministic
and independent of the batch split, R14; grad_input with deterministic=True)."""
import pytest
import torch

import synth
import paper_2401_06197_b200 as pkg
from paper_2401_06197_b200.pipeline import HostPipeline

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chunks", [1, 3, 5])
def test_pipeline_matches_direct_calls(chunks, cuda_device):
    N, H, W, G, D = 5, 9, 11, 4, 16
    x, om, gy = synth.make_case(N, H, W, G, D, H, W, 9, 3 * G * 9, "f32")
    hx, hom, hgy = x.pin_memory(), om.pin_memory(), gy.pin_memory()
    hy, hgx, hgom = (torch.empty_like(t).pin_memory() for t in (x, x, om))
    dx, dom_, dgy = (torch.empty_like(t, device=cuda_device) for t in (x, om, gy))
    dy, dgx, dgom = (torch.empty_like(t, device=cuda_device) for t in (x, x, om))
    b = [(c * N // chunks, (c + 1) * N // chunks) for c in range(chunks)]

    def cin(c):
        lo, hi = b[c]
        for d, h in ((dx, hx), (dom_, hom), (dgy, hgy)):
            d[lo:hi].copy_(h[lo:hi], non_blocking=True)

    def comp(c):
        lo, hi = b[c]
        pkg.forward(dx[lo:hi], dom_[lo:hi], group=G, out=dy[lo:hi])
        pkg.backward(dx[lo:hi], dom_[lo:hi], dgy[lo:hi], group=G, grad_input=dgx[lo:hi],
                     grad_offset_mask=dgom[lo:hi], deterministic=True)

    def cout(c):
        lo, hi = b[c]
        for h, d in ((hy, dy), (hgx, dgx), (hgom, dgom)):
            h[lo:hi].copy_(d[lo:hi], non_blocking=True)

    pipe = HostPipeline(cuda_device, chunks)
    for _ in range(2):  # a second pass exercises the cross-pass event ordering
        start, end = pipe.run(cin, comp, cout)
    torch.cuda.synchronize()
    assert end.elapsed_time(start) <= 0 or start.elapsed_time(end) >= 0
    xd, omd, gyd = x.to(cuda_device), om.to(cuda_device), gy.to(cuda_device)
    y = pkg.forward(xd, omd, group=G)
    gx, gom = pkg.backward(xd, omd, gyd, group=G, deterministic=True)
    torch.cuda.synchronize()
    assert torch.equal(hy, y.cpu())
    assert torch.equal(hgom, gom.cpu())
    assert torch.equal(hgx, gx.cpu())
