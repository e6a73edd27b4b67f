"""Module-path measurement on one B200: the fused offset/mask linear
 on tcgen05 tensor cores, and the lightweight module forward (linear + DCNv4
forward), over the c2 (224^2, batch 64) or c3 (800x1280, batch 8) stage
shapes in f16/bf16.

Per stage: linear us, its algorithmic bytes (x read + W read + om write) and flops
(2*R*C*J), GB/s and TFLOP/s against MEASURED_PEAKS.json, and the module forward us.
K reps of each call are captured in one CUDA graph with event nodes between calls.
One JSON line per run.

  python scripts/bench_module.py [--workload c2|c3] [--dtype f16|bf16] [--reps 20]
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
from paper_2401_06197_b200 import binding, module  # noqa: E402

STAGES = {"c2": (64, [(56, 56, 64, 4), (28, 28, 128, 8), (14, 14, 256, 16), (7, 7, 512, 32)]),
          "c3": (8, [(200, 320, 64, 4), (100, 160, 128, 8), (50, 80, 256, 16), (25, 40, 512, 32)])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=list(STAGES))
    ap.add_argument("--dtype", default="f16", choices=["f16", "bf16"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--weights", default="synth", choices=["synth", "zero"],
                    help="zero: W = 0, b = 0 (om = 0: zero offsets and masks; ablation)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    N, shapes = STAGES[args.workload]
    N = args.batch or N
    peak_bw, src = bench._peaks()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak_tf = float(json.load(f)["bf16_tflops"])
    except Exception:
        peak_tf = 2250.0
    rows = []
    stream = torch.cuda.Stream(device=dev)
    for H, W, C, G in shapes:
        K = 9
        S = module.om_stride_for(G, K)
        x, _, _ = synth.make_case(N, H, W, G, C // G, H, W, K, 3 * G * K, args.dtype, with_gy=False)
        w, b = synth.make_linear(C, G, K, args.dtype)
        if args.weights == "zero":
            w, b = torch.zeros_like(w), torch.zeros_like(b)
        xd, wd, bd = x.to(dev), w.to(dev), b.to(dev)
        om = torch.empty((N, H, W, S), dtype=xd.dtype, device=dev)
        y = torch.empty_like(xd)
        y2 = torch.empty_like(xd)
        calls = [("linear", lambda: module.offset_mask_linear(xd, wd, bd, G, S, out=om)),
                 ("dcnv4_fwd", lambda: binding.forward(xd, om, G, out=y)),
                 ("fused", lambda: module.forward_fused(xd, wd, bd, G, out=y2))]
        with torch.cuda.stream(stream):
            for _ in range(3):
                for _, fn in calls:
                    fn()
        stream.synchronize()
        nc = len(calls)
        evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(nc * args.reps + 1)]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            evs[0].record(stream)
            i = 1
            for _ in range(args.reps):
                for _, fn in calls:
                    fn()
                    evs[i].record(stream)
                    i += 1
        with torch.cuda.stream(stream):
            graph.replay()
        torch.cuda.synchronize()
        med = [sorted(evs[nc * r + c].elapsed_time(evs[nc * r + c + 1]) for r in range(args.reps))[args.reps // 2]
               for c in range(nc)]
        lin, dcn, fus = med
        same = torch.mean((y == y2).double()).item()
        R, J = N * H * W, 3 * G * K
        by = (R * C + J * C + R * S) * 2
        fl = 2.0 * R * C * J
        rows.append({"shape": f"{H}x{W}x{C} G{G}", "N": N, "S": S,
                     "linear_us": round(lin * 1e3, 2), "linear_alg_bytes": by,
                     "linear_GBs": round(by / lin / 1e6, 1), "linear_frac_hbm": round(by / lin / 1e6 / peak_bw, 4),
                     "linear_TFLOPs": round(fl / lin / 1e9, 1), "linear_frac_tc": round(fl / lin / 1e9 / peak_tf, 4),
                     "dcnv4_fwd_us": round(dcn * 1e3, 2), "module_us": round((lin + dcn) * 1e3, 2),
                     "fused_us": round(fus * 1e3, 2), "fused_vs_two_call_bit_equal": round(same, 5)})
        del graph
    tot = sum(r["fused_us"] for r in rows)
    tot2 = sum(r["module_us"] for r in rows)
    line = {"metric": "DCNv4 lightweight module forward: fused kernel (value) vs linear + dcnv4_forward (two_call)",
            "value": round(N / (tot * 1e-6), 2), "unit": "imgs/s",
            "two_call_imgs_s": round(N / (tot2 * 1e-6), 2), "n_gpus": 1, "dtype": args.dtype,
            "data": "synthetic", "config": {"workload": f"module_{args.workload}", "batch": N, "reps": args.reps, "weights": args.weights,
                                            "l2": "per-stage working sets up to 0.2 GB; no flush"},
            "peaks": {"hbm_gbs": peak_bw, "tc_tflops": peak_tf, "source": src}, "stages": rows}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
