"""Small runs of the round-2 kernels for compute-sanitizer: the reworked bwd33 (fp32 8-B and
half 4-B bin entries, distributed P1, direct grad_offset_mask stores), the grouped forward,
the tcgen05 GEMMs (K-/MN-major, two segments, split-K, 3xTF32) and the full module."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2401_06197_b200 as pkg  # noqa: E402
from paper_2401_06197_b200 import module as mod  # noqa: E402

dev = torch.device("cuda:0")
for dt in ("f32", "f16", "bf16"):
    x, om, gy = synth.make_case(2, 17, 13, 4, 16, 17, 13, 9, 108, dt)
    x, om, gy = x.to(dev), om.to(dev), gy.to(dev)
    pkg.backward(x, om, gy, group=4)
    pkg.backward(x, om, gy, group=4, softmax=True)
    x2, om2, _ = synth.make_case(1, 9, 7, 8, 16, 9, 7, 9, 216, dt, with_gy=False)
    pkg.forward_grouped([x, x2.to(dev)], [om, om2.to(dev)], [4, 8])
    prm = {k: v.to(dev) for k, v in synth.make_module_params(64, 4, 9, dt).items()}
    y, saved = mod.full_forward(x, prm, 4)
    mod.full_backward(x, prm, 4, gy, saved)
torch.cuda.synchronize()
print("sanitize_r2 done")
