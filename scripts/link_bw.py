"""Host<->device link bandwidth on this box (pinned buffers): H2D alone, D2H alone, both
concurrently on two streams.  Context for the e2e numbers (bench.py)."""
import torch
n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); 
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / 1e3
def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
for name, fn, by in (("h2d", h2d, n), ("d2h", d2h, n), ("both", both, 2 * n)):
    print(name, round(by / t(fn) / 1e9, 1), "GB/s")
