"""Small fwd + bwd runs over every kernel path (TMA-halo kernels, global-gather fallback,
out-of-halo fallback, half dtypes, softmax) for compute-sanitizer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2401_06197_b200 as pkg  # noqa: E402

dev = torch.device("cuda:0")
cases = [
    # (N, H, W, G, D, dtype, kernel, stride, pad, dilation, scale, offsets, softmax)
    (2, 9, 11, 2, 16, "f32", 3, 1, 1, 1, 1.0, "u2", False),
    (1, 12, 10, 4, 16, "f16", 3, 1, 1, 1, 1.0, "u8", False),
    (1, 10, 9, 4, 16, "bf16", 3, 1, 1, 1, 0.5, "u2", True),
    (2, 9, 8, 2, 16, "f32", 3, 2, 1, 2, 1.0, "u2", False),
    (1, 7, 7, 2, 32, "f32", 5, 1, 2, 1, 1.0, "u8", False),
    (1, 6, 5, 3, 8, "f16", 3, 1, 1, 1, 1.0, "u2", False),
]
for (N, H, W, G, D, dt, k, st, pd, dl, sc, off, sm) in cases:
    p = pkg.make_params(N, H, W, G, D, k, st, pd, dl, sc)
    Ho, Wo = pkg.output_size(p)
    x, om, gy = synth.make_case(N, H, W, G, D, Ho, Wo, k * k, 3 * G * k * k, dt, offsets=off)
    x, om, gy = x.to(dev), om.to(dev), gy.to(dev)
    kw = dict(group=G, kernel_size=k, stride=st, pad=pd, dilation=dl, offset_scale=sc, softmax=sm)
    y = pkg.forward(x, om, **kw)
    gx, gom = pkg.backward(x, om, gy, **kw)
    gxd, _ = pkg.backward(x, om, gy, deterministic=True, **kw)  # int64 fixed-point path
    torch.cuda.synchronize()
    print("ok", (N, H, W, G, D, dt, k, st, pd, dl, sc, off, sm), float(y.float().abs().sum()),
          float(gx.float().abs().sum()), float(gom.float().abs().sum()),
          float(gxd.float().abs().sum()))

# module path (NEXT-2): tcgen05 linear and the fused module forward (TMA, mbarriers, TMEM)
from paper_2401_06197_b200 import module, msda  # noqa: E402

for (N, H, W, G, D, dt) in [(1, 20, 13, 8, 16, "f16"), (1, 9, 11, 2, 64, "bf16"), (2, 7, 9, 4, 16, "f16")]:
    C = G * D
    x, _, _ = synth.make_case(N, H, W, G, D, H, W, 9, 27 * G, dt, with_gy=False)
    w, b = synth.make_linear(C, G, 9, dt)
    x, w, b = x.to(dev), w.to(dev), b.to(dev)
    om = module.offset_mask_linear(x, w, b, G)
    y = module.forward_fused(x, w, b, G)
    torch.cuda.synchronize()
    print("ok module", (N, H, W, G, D, dt), float(om.float().abs().sum()), float(y.float().abs().sum()))

# MSDA (NEXT-3): forward, 16-B backward (f32) and 8-B half backward
shapes = ((6, 8), (3, 4), (2, 2))
for dt in ("f32", "bf16"):
    S = sum(h * w for h, w in shapes)
    value, loc, attn, gout = synth.make_msda_case(2, 11, 2, 32, 3, shapes, dt)
    value, loc, attn, gout = (t.to(dev) for t in (value, loc, attn, gout))
    out = msda.forward(value, loc, attn, shapes)
    gv, gl, ga = msda.backward(value, loc, attn, gout, shapes)
    torch.cuda.synchronize()
    print("ok msda", dt, float(out.float().abs().sum()), float(gv.float().abs().sum()))
