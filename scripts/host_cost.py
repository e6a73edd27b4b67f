import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, synth
from paper_2401_06197_b200 import module, binding
dev = torch.device("cuda:0")
x, om, _ = synth.make_case(8, 56, 56, 4, 16, 56, 56, 9, 108, "f16", with_gy=False)
w, b = synth.make_linear(64, 4, 9, "f16")
x, om, w, b = x.to(dev), om.to(dev), w.to(dev), b.to(dev)
for name, fn in [("forward_fused", lambda: module.forward_fused(x, w, b, 4)),
                 ("offset_mask_linear", lambda: module.offset_mask_linear(x, w, b, 4)),
                 ("dcnv4 forward", lambda: binding.forward(x, om, 4))]:
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(name, "host us/call", (t1 - t0) / 20 * 1e6, "total us/call", (t2 - t0) / 20 * 1e6)
