"""Sweep launch knobs (chunks per lane, CTA tile) on the bench stage shapes; prints one
JSON line per (stage, pass, knob) with the median CUDA-event time and algorithmic GB/s.
The library reads its ablation switches once per process (csrc/ablation.h), so every knob
combination runs in a child process with its switches in the environment.

  python scripts/tune.py --workload c4 [--cpl 1,2,4] [--tiles "8,8,2;4,8,4"] [--reps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_2401_06197_b200 as pkg  # noqa: E402


def timeit(fn, reps):
    """Average GPU time per call: `reps` calls captured in one CUDA graph (no host launch
    overhead in the measurement), replayed 3 times; the best replay is reported."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(reps):
            fn()
    best = 1e30
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            graph.replay()
            b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--cpl", default="")
    ap.add_argument("--tiles", default="")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--stages", default="")
    ap.add_argument("--offsets", default="u2")
    ap.add_argument("--passes", default="fwd,bwd")
    ap.add_argument("--child", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if not args.child:
        import subprocess
        for cpl in (args.cpl.split(",") if args.cpl else [""]):
            for tile in (args.tiles.split(";") if args.tiles else [""]):
                env = dict(os.environ, DCNV4_FWD_CPL=cpl, DCNV4_BWD_CPL=cpl, DCNV4_TILE=tile)
                argv = [a for a in sys.argv[1:]]
                subprocess.run([sys.executable, os.path.abspath(__file__), *argv, "--child"],
                               env=env, check=True)
        return
    cfg = bench.WORKLOADS[args.workload]
    N = args.batch or cfg["batch"]
    peak, _ = bench._peaks()
    tile = os.environ.get("DCNV4_TILE", "")
    stages = [int(s) for s in args.stages.split(",")] if args.stages else range(len(cfg["stages"]))
    dev = torch.device("cuda:0")
    for si in stages:
        H, W, G, D = cfg["stages"][si]
        x, om, gy = synth.make_case(N, H, W, G, D, H, W, 9, 27 * G, cfg["dtype"], offsets=args.offsets)
        x, om, gy = x.to(dev), om.to(dev), gy.to(dev)
        y, gx, gom = torch.empty_like(x), torch.empty_like(x), torch.empty_like(om)
        ws = torch.empty(max(16, pkg.workspace_bytes(pkg.make_params(N, H, W, G, D), x.dtype)),
                         dtype=torch.uint8, device=dev)
        for ps in args.passes.split(","):
            if ps == "bwd" and not cfg["backward"]:
                continue
            if ps == "fwd":
                fn = lambda: pkg.forward(x, om, group=G, out=y)  # noqa: E731
            else:
                fn = lambda: pkg.backward(x, om, gy, group=G, grad_input=gx,  # noqa: E731
                                          grad_offset_mask=gom, workspace=ws)
            ms = timeit(fn, args.reps)
            b = bench._alg_bytes(x, om, ps == "bwd")
            li = pkg.launch_info(pkg.make_params(N, H, W, G, D), x.dtype, ps == "bwd")
            print(json.dumps({"stage": f"{H}x{W}x{G * D} G{G} D{D}", "N": N, "dtype": cfg["dtype"],
                              "pass": ps, "cpl": li["chunks_per_lane"], "tile_env": tile,
                              "threads": li["threads_per_cta"], "pix_per_cta": li["pixels_per_cta"],
                              "us": round(ms * 1e3, 1), "GBs": round(b / ms / 1e6, 1),
                              "frac": round(b / ms / 1e6 / peak, 4)}), flush=True)
        del x, om, gy, y, gx, gom, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
