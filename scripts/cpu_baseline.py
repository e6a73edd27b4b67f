"""CPU baseline protocol of SURVEY 8(d).4 / BASELINE.md section 4: the fp64 C oracle as it
stands (plain scalar C, OpenMP over (image, group)), timed on THIS machine's host cores for
every BASELINE config, forward and backward separately, with 1 thread and with nproc
threads.  Each measurement runs a bounded sample of images (the oracle's cost is linear
in the image count) and reports per-image milliseconds and images/s; the wall-clock
median of 3 runs (1 run when one run exceeds 10 s).  The thread count is fixed per child
process (OpenMP reads OMP_NUM_THREADS at library load).

  python scripts/cpu_baseline.py [--out profiles/r02_cpu_baseline.json]
"""
import argparse
import json
import os
import platform
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = [  # (name, stages (H, W, G, D), dtype, batch, backward)
    ("c2_f32", [(56, 56, 4, 16), (28, 28, 8, 16), (14, 14, 16, 16), (7, 7, 32, 16)], "f32", 64, False),
    ("c2_f16", [(56, 56, 4, 16), (28, 28, 8, 16), (14, 14, 16, 16), (7, 7, 32, 16)], "f16", 64, False),
    ("c3_f16", [(200, 320, 4, 16), (100, 160, 8, 16), (50, 80, 16, 16), (25, 40, 32, 16)], "f16", 8, False),
    ("c4", [(56, 56, 4, 16), (28, 28, 8, 16), (14, 14, 16, 16), (7, 7, 32, 16)], "f32", 512, True),
    ("c5_bf16", [(64, 64, 20, 16), (32, 32, 40, 16), (16, 16, 80, 16)], "bf16", 32, True),
]

CHILD = r'''
import json, sys, time
sys.path.insert(0, %(root)r)
import oracle, synth
stages, dtype, nimg, backward = %(stages)r, %(dtype)r, %(nimg)d, %(backward)r
data = []
for H, W, G, D in stages:
    g = oracle.Geometry(N=nimg, H=H, W=W, G=G, D=D)
    x, om, gy = synth.make_case(nimg, H, W, G, D, H, W, 9, 27 * G, dtype)
    data.append((g, oracle._f64(x), oracle._f64(om), oracle._f64(gy)))
out = {}
for kind in (("fwd", "bwd") if backward else ("fwd",)):
    runs = []
    for r in range(3):
        t0 = time.perf_counter()
        for g, x, om, gy in data:
            if kind == "fwd":
                oracle.forward(g, x, om)
            else:
                oracle.backward(g, x, om, gy)
        runs.append(time.perf_counter() - t0)
        if runs[-1] > 10.0:
            break
    runs.sort()
    out[kind] = runs[len(runs) // 2]
print(json.dumps(out))
'''


def lscpu():
    info = {}
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in txt.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "CPU(s)", "Thread(s) per core", "Core(s) per socket"):
                info[k.strip()] = v.strip()
    except Exception as e:  # noqa: BLE001
        info["error"] = repr(e)
    return info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cpu_baseline.json"))
    ap.add_argument("--budget", type=float, default=4.0, help="target seconds per (config, threads) sample")
    args = ap.parse_args()
    import oracle
    oracle.build()
    nproc = len(os.sched_getaffinity(0))
    rows = []
    for name, stages, dtype, batch, backward in CONFIGS:
        for threads in (1, nproc):
            env = dict(os.environ, OMP_NUM_THREADS=str(threads))
            # probe one image to size the sample
            probe = CHILD % dict(root=ROOT, stages=stages, dtype=dtype, nimg=1, backward=backward)
            t1 = json.loads(subprocess.run([sys.executable, "-c", probe], env=env, capture_output=True,
                                           text=True, check=True).stdout)
            per = sum(t1.values())
            nimg = max(1, min(batch, int(args.budget / max(per, 1e-3))))
            code = CHILD % dict(root=ROOT, stages=stages, dtype=dtype, nimg=nimg, backward=backward)
            t = json.loads(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                          text=True, check=True).stdout)
            row = {"config": name, "dtype": dtype, "batch": batch, "threads": threads, "sample_images": nimg}
            for kind, sec in t.items():
                row[f"{kind}_ms_per_image"] = round(1e3 * sec / nimg, 3)
                row[f"{kind}_imgs_per_s"] = round(nimg / sec, 2)
                row[f"{kind}_s_full_batch"] = round(sec / nimg * batch, 2)
            rows.append(row)
            print(json.dumps(row), flush=True)
    res = {"machine": {"nproc": nproc, "lscpu": lscpu(), "python": platform.python_version()},
           "oracle": "oracle/dcnv4_oracle.c, gcc -O2 -fopenmp -ffp-contract=off, fp64 scalar, OpenMP over (n, g)",
           "protocol": "SURVEY 8(d).4: 1 thread and nproc threads, forward and backward separately, "
                       "median of 3 runs (1 when a run exceeds 10 s), bounded image sample scaled to the batch",
           "rows": rows}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
