"""Run one stage shape of a bench workload a few times (for ncu captures).

  python scripts/profile_stage.py --workload c4 --stage 0 [--reps 3] [--fwd-only]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2401_06197_b200 as pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--stage", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--fwd-only", action="store_true")
    ap.add_argument("--offsets", default="u2")
    args = ap.parse_args()
    cfg = bench.WORKLOADS[args.workload]
    H, W, G, D = cfg["stages"][args.stage]
    N = args.batch or cfg["batch"]
    dev = torch.device("cuda:0")
    x, om, gy = synth.make_case(N, H, W, G, D, H, W, 9, 27 * G, cfg["dtype"],
                                offsets=args.offsets)
    x, om, gy = x.to(dev), om.to(dev), gy.to(dev)
    y = torch.empty_like(x)
    gx = torch.empty_like(x)
    gom = torch.empty_like(om)
    for _ in range(args.reps):
        pkg.forward(x, om, group=G, out=y)
        if cfg["backward"] and not args.fwd_only:
            pkg.backward(x, om, gy, group=G, grad_input=gx, grad_offset_mask=gom)
    torch.cuda.synchronize()
    print("launch info fwd", pkg.launch_info(pkg.make_params(N, H, W, G, D), x.dtype))
    print("launch info bwd", pkg.launch_info(pkg.make_params(N, H, W, G, D), x.dtype, True))


if __name__ == "__main__":
    main()
