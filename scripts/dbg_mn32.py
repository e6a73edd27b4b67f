"""Debug: fp32 MN-major GEMM operand layout (grad_input with identity / permutation weights)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_06197_b200 import module as mod
dev = torch.device("cuda:0")
torch.manual_seed(0)
for dt in (torch.float16, torch.float32):
    M, K = 256, 64
    gy = torch.randn(M, K, device=dev).to(dt)
    W = torch.eye(K, device=dev).to(dt)
    gx = mod.linear_grad_input(gy, W)
    torch.cuda.synchronize()
    err = (gx.float() - gy.float()).abs()
    print(dt, "identity: max err", err.max().item())
    if err.max() > 1e-3:
        # which source column does each output column come from?
        for c in range(0, 64, 4):
            col = gx[:, c].float()
            best = ((gy.float() - col[:, None]).abs().sum(0)).argmin().item()
            print("  out col", c, "<- gy col", best, "err", ((gy[:, best].float() - col).abs().max().item()))
    # weight grad: dW = gy^T x with x = identity rows (M = K): dW = gy^T
    x = torch.eye(M, K, device=dev).to(dt)
    gw, _ = mod.linear_grad_weight(x, gy, with_bias=False)
    torch.cuda.synchronize()
    ref = gy.float().t() @ x.float()
    e2 = (gw.float() - ref).abs()
    print(dt, "wgrad err", e2.max().item())
    if e2.max() > 1e-3:
        for r in range(0, 64, 8):
            row = gw[r].float()
            best = ((ref - row[None, :]).abs().sum(1)).argmin().item()
            print("  out row", r, "<- ref row", best)
