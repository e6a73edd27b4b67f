import os, sys, torch, threading
sys.path.insert(0, '.')
import synth, paper_2401_06197_b200 as pkg
from paper_2401_06197_b200 import binding as b
dev = torch.device('cuda:0')
N,H,W,G = 2,9,9,2
x, om, gy = (t.to(dev) for t in synth.make_case(N, H, W, G, 16, H, W, 9, 27*G, 'f32'))
orig = b.backward
def spy(x, om, gy, *a, **k):
    print('thread', threading.current_thread().name, 'ptr%16', x.data_ptr()%16, om.data_ptr()%16, gy.data_ptr()%16, gy.is_contiguous(), gy.stride(), a, k)
    return orig(x, om, gy, *a, **k)
b.backward = spy
xr = x.clone().requires_grad_(True); omr = om.clone().requires_grad_(True)
y = pkg.dcnv4(xr, omr, G); y.backward(gy)
gx, gom = orig(x, om, gy, group=G)
print('diffs', int((omr.grad != gom).sum()))
# direct call from a worker thread
res = {}
def work():
    res['g'] = orig(x, om, gy, group=G)
th = threading.Thread(target=work); th.start(); th.join()
print('thread vs main diffs', int((res['g'][1] != gom).sum()))
