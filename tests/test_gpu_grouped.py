"""dcnv4_forward_grouped (include/dcnv4.h): several independent forwards in one persistent
launch must equal the per-problem dcnv4_forward bit for bit (same arithmetic per output),
fall back to one launch per problem when the problems cannot share a kernel, skip empty
problems, and validate every problem before launching (errors name the index)."""
import pytest
import torch

import oracle
import synth
import paper_2401_06197_b200 as pkg

pytestmark = pytest.mark.gpu

C2 = [(56, 56, 4), (28, 28, 8), (14, 14, 16), (7, 7, 32)]
C3 = [(200, 320, 4), (100, 160, 8), (50, 80, 16), (25, 40, 32)]


def _case(N, H, W, G, D, dtype, offsets="u2", images=None):
    x, om, _ = synth.make_case(N, H, W, G, D, H, W, 9, 27 * G, dtype, with_gy=False, offsets=offsets,
                               images=images)
    dev = torch.device("cuda:0")
    return x.to(dev), om.to(dev)


@pytest.mark.parametrize("dtype", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("shapes,N", [(C2, 3), (C3, 1), ([(9, 13, 4), (5, 6, 8), (17, 3, 4)], 2)],
                         ids=["c2", "c3_b1", "ragged"])
def test_grouped_equals_separate(dtype, shapes, N):
    cases = [_case(N, H, W, G, 16, dtype, images=list(range(i, i + N))) for i, (H, W, G) in enumerate(shapes)]
    xs, oms = [c[0] for c in cases], [c[1] for c in cases]
    groups = [G for _, _, G in shapes]
    ys = pkg.forward_grouped(xs, oms, groups)
    for x, om, G, y in zip(xs, oms, groups, ys):
        assert torch.equal(y, pkg.forward(x, om, group=G))


def test_grouped_against_oracle_and_u8():
    shapes = [(14, 14, 4), (7, 7, 8)]
    cases = [_case(1, H, W, G, 16, "f32", offsets="u8") for H, W, G in shapes]
    ys = pkg.forward_grouped([c[0] for c in cases], [c[1] for c in cases], [G for _, _, G in shapes])
    for (H, W, G), (x, om), y in zip(shapes, cases, ys):
        g = oracle.Geometry(N=1, H=H, W=W, G=G, D=16)
        ref, ra = oracle.forward(g, x.cpu(), om.cpu(), with_abs=True)
        assert oracle.abs_scaled_error(y.cpu(), ref, ra) <= 1e-5


def test_grouped_fallback_mixed_layouts_and_empty():
    """D = 16 and D = 32 need different kernel instantiations: one launch each, same
    results; an empty batch is skipped."""
    x1, om1 = _case(2, 12, 12, 4, 16, "f16")
    x2, om2 = _case(2, 10, 9, 4, 32, "f16")
    x3, om3 = _case(0, 8, 8, 4, 16, "f16")
    ys = pkg.forward_grouped([x1, x2, x3], [om1, om2, om3], [4, 4, 4])
    assert torch.equal(ys[0], pkg.forward(x1, om1, group=4))
    assert torch.equal(ys[1], pkg.forward(x2, om2, group=4))
    assert ys[2].shape[0] == 0


def test_grouped_validation_names_the_problem():
    x1, om1 = _case(1, 8, 8, 4, 16, "f32")
    bad = om1[..., :-1].contiguous()
    with pytest.raises((pkg.DCNv4Error, ValueError)):
        pkg.forward_grouped([x1, x1], [om1, bad], [4, 4])
