import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
from paper_2401_06197_b200 import msda
dev = torch.device("cuda:0")
g = oracle.MSDAGeometry(N=2, Lq=12, M=5, D=4, P=1, shapes=((9, 7), (3, 10), (4, 6), (4, 4)))
value, loc, attn, gout = synth.make_msda_case(g.N, g.Lq, g.M, g.D, g.P, g.shapes, "f32")
vd, ld, ad, gd = (t.to(dev) for t in (value, loc, attn, gout))
gv, gl, ga = msda.backward(vd, ld, ad, gd, g.shapes)
out = msda.forward(vd, ld, ad, g.shapes)
torch.cuda.synchronize()
rgv, rgl, rga, agv, agl, aga = oracle.msda_backward(g, value, loc, attn, gout, with_abs=True)
ref = oracle.msda_forward(g, value, loc, attn)
for name, gpu, r, a in (("gattn", ga, rga, aga), ("gloc", gl, rgl, agl), ("gval", gv, rgv, agv)):
    gpu = gpu.double().cpu().numpy()
    e = np.abs(gpu - r) / (a + 1e-30)
    idx = np.unravel_index(np.argmax(e), e.shape)
    print(name, "max e", e.max(), "at", idx, "gpu", gpu[idx], "ref", r[idx], "abs", a[idx])
    print("   count > 1e-5:", int((e > 1e-5).sum()), "of", e.size)
i = np.unravel_index(np.argmax(np.abs(ga.double().cpu().numpy() - rga) / (aga + 1e-30)), rga.shape)
n, q, m, l, p = i
print("loc", loc[n, q, m, l, p].tolist(), "attn", float(attn[n, q, m, l, p]), "shape", g.shapes[l])
H, W = g.shapes[l]
print("pix", float(loc[n, q, m, l, p, 0]) * W - 0.5, float(loc[n, q, m, l, p, 1]) * H - 0.5)
print("out err", np.abs(out.double().cpu().numpy() - ref).max())
