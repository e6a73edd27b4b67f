#!/usr/bin/env python
"""bench.py -- DCNv4 spatial aggregation on B200: the driver's benchmark contract.

Default workload (BASELINE.json configs[3], "c4"): one training step of the DCNv4 core
operator over the four InternImage-T 224^2 stage shapes (56^2x64 G4, 28^2x128 G8,
14^2x256 G16, 7^2x512 G32; D=16), fp32, forward + backward (every SURVEY.md 8(a) row),
global batch 512 sharded by batch over the ranks (strong scaling, no collective on the
data path).  Inputs are seeded synthetic tensors (synth/)
resident in HBM.

Timed region: K steps captured in CUDA graphs with external event nodes between the
library calls, replayed between a barrier + synchronize on both sides; the step time is
the max over ranks.  Per-call durations come from those event nodes (on the launching
stream), giving the per-stage table and the roofline of the dominant kernel.  When a
step's working set is below 2x L2 a 2xL2 buffer is written after every step (timed by its
own events and excluded), so no step reads inputs another step left in L2.

The default run also measures the forward sweeps (c2, c3 at batch 1 and 8, the paper-
comparable D=32 shape sets c2'/c3' next to the A100 rows of P:304-305 / P:362-363, and
c5) and reports them under "forward_sweeps" (--no-extras skips them).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
  python bench.py --impl reference ...   # the fp64 CPU oracle as the reference arm
--gpus N > 1 outside torchrun re-launches itself under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# OpenMP of the oracle (cpu_baseline / reference arm) reads this at library load.
os.environ.setdefault("OMP_NUM_THREADS", str(len(os.sched_getaffinity(0))))

METRIC = ("DCNv4 fwd/bwd µs and HBM GB/s (% of B200 peak) per stage shape; "
          "imgs/s at 1/2/4/8 GPU")
# stage shapes (H, W, G, D)
STAGES_224 = [(56, 56, 4, 16), (28, 28, 8, 16), (14, 14, 16, 16), (7, 7, 32, 16)]
STAGES_800 = [(200, 320, 4, 16), (100, 160, 8, 16), (50, 80, 16, 16), (25, 40, 32, 16)]
STAGES_UNET = [(64, 64, 20, 16), (32, 32, 40, 16), (16, 16, 80, 16)]
# Tab. op_low_res and Tab. op_high_res: group dim 32,
# batch 64 / 1; the A100 DCNv4 rows (ms, fp32 / fp16) for context
STAGES_LOW_D32 = [(56, 56, 4, 32), (28, 28, 8, 32), (14, 14, 16, 32), (7, 7, 32, 32), (14, 14, 24, 32)]
STAGES_HIGH_D32 = [(200, 320, 4, 32), (100, 160, 8, 32), (50, 80, 16, 32), (25, 40, 32, 32),
                   (64, 64, 24, 32)]
PAPER_A100_MS = {
    "low": {"f32": [0.606, 0.303, 0.145, 0.0730, 0.224], "f16": [0.404, 0.230, 0.123, 0.0680, 0.147]},
    "high": {"f32": [0.210, 0.124, 0.0707, 0.0452, 0.103], "f16": [0.136, 0.0895, 0.0589, 0.0426, 0.0672]},
}
WORKLOADS = {
    "c1": dict(desc="BASELINE configs[0]: tiny 8x8x32 G2 D16 fp32 fwd+bwd (parity case)",
               stages=[(8, 8, 2, 16)], dtype="f32", batch=1, backward=True, shard=True),
    "c4": dict(desc="BASELINE configs[3]: training fwd+bwd, InternImage-T 224^2 four-stage "
                    "shapes, D=16, fp32, global batch 512 sharded by batch",
               stages=STAGES_224, dtype="f32", batch=512, backward=True, shard=True),
    "c2_f32": dict(desc="BASELINE configs[1]: 224^2 stage sweep, D=16, fp32 forward, batch 64",
                   stages=STAGES_224, dtype="f32", batch=64, backward=False, shard=False),
    "c2_f16": dict(desc="BASELINE configs[1]: 224^2 stage sweep, D=16, fp16 forward, batch 64",
                   stages=STAGES_224, dtype="f16", batch=64, backward=False, shard=False),
    "c3_f16": dict(desc="BASELINE configs[2]: 800x1280 FlashInternImage stages, D=16, fp16 "
                        "forward, batch 8", stages=STAGES_800, dtype="f16", batch=8,
                   backward=False, shard=False),
    "c5_bf16": dict(desc="BASELINE configs[4]: U-Net 64^2 latents C=320/640/1280, D=16, bf16 "
                         "fwd+bwd, batch 32", stages=STAGES_UNET, dtype="bf16", batch=32,
                    backward=True, shard=False),
    "c2p_f32": dict(desc="c2' (SURVEY 8(d).1): Tab. op_low_res shapes, D=32, fp32 forward, batch 64",
                    stages=STAGES_LOW_D32, dtype="f32", batch=64, backward=False, shard=False,
                    paper="low"),
    "c2p_f16": dict(desc="c2' (SURVEY 8(d).1): Tab. op_low_res shapes, D=32, fp16 forward, batch 64",
                    stages=STAGES_LOW_D32, dtype="f16", batch=64, backward=False, shard=False,
                    paper="low"),
    "c3p_f32": dict(desc="c3' (SURVEY 8(d).1): Tab. op_high_res shapes, D=32, fp32 forward, batch 1",
                    stages=STAGES_HIGH_D32, dtype="f32", batch=1, backward=False, shard=False,
                    paper="high"),
    "c3p_f16": dict(desc="c3' (SURVEY 8(d).1): Tab. op_high_res shapes, D=32, fp16 forward, batch 1",
                    stages=STAGES_HIGH_D32, dtype="f16", batch=1, backward=False, shard=False,
                    paper="high"),
    # all stages of one step in ONE persistent launch (dcnv4_forward_grouped)
    "c3_f16_grouped": dict(desc="BASELINE configs[2] stages, D=16, fp16 forward, batch 8, the four "
                                "stages in one dcnv4_forward_grouped launch", stages=STAGES_800,
                           dtype="f16", batch=8, backward=False, shard=False, grouped=True),
    "c2_f16_grouped": dict(desc="BASELINE configs[1] stages, D=16, fp16 forward, batch 64, the four "
                                "stages in one dcnv4_forward_grouped launch", stages=STAGES_224,
                           dtype="f16", batch=64, backward=False, shard=False, grouped=True),
    # NEXT-2 (R21): the lightweight DCNv4 module forward, one fused kernel per
    # stage (offset/mask linear on tcgen05 + aggregation; om never leaves the SM)
    "module_c2": dict(desc="NEXT-2 fused lightweight module forward (P:334, P:1003-1009) on the "
                           "224^2 stage shapes, D=16, fp16, batch 64", stages=STAGES_224,
                      dtype="f16", batch=64, backward=False, shard=False, module=True),
    "module_c3": dict(desc="NEXT-2 fused lightweight module forward on the 800x1280 stage "
                           "shapes, D=16, fp16, batch 8", stages=STAGES_800, dtype="f16", batch=8,
                      backward=False, shard=False, module=True),
    # NEXT-2, full module (R22): input projection, fused om-linear + aggregation sampling
    # the projection, output projection; backward = every GEMM's grads + DCNv4 backward
    "module_full_c2": dict(desc="NEXT-2 full DCNv4 module (1x1 in/out projections, P:198, "
                                "P:1006-1009) forward, 224^2 stage shapes, D=16, fp16, batch 64",
                           stages=STAGES_224, dtype="f16", batch=64, backward=False, shard=False,
                           module="full"),
    "module_full_train_c2": dict(desc="NEXT-2 full DCNv4 module forward + backward (all weight and "
                                      "input gradients), 224^2 stage shapes, D=16, fp16, batch 64",
                                 stages=STAGES_224, dtype="f16", batch=64, backward=True, shard=False,
                                 module="full"),
}
# forward sweeps measured by the default run (workload, batch override)
EXTRAS = [("c2_f32", None), ("c2_f16", None), ("c2_f16_grouped", None), ("c3_f16", 1),
          ("c3_f16_grouped", 1), ("c3_f16", 8), ("c3_f16_grouped", 8), ("c2p_f32", None),
          ("c2p_f16", None), ("c3p_f32", None), ("c3p_f16", None), ("c5_bf16", None)]
K = 9
MIN_TIMED_S = 0.4      # auto step count: timed region >= this (>= 2 clock samples at 50 ms)
GRAPH_STEPS = 100      # steps per captured graph (longer regions replay it)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def shape_name(H, W, G, D):
    return f"{H}x{W}x{G * D} G{G} D{D}"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    FIELDS = ("uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid: str | None):
        self.uuid = uuid
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            if self.uuid and parts[0] != self.uuid:
                continue
            self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0,
                    "samples_in_timed_region": 0}
        inside = [s for t, s in self.samples if t0 <= t <= t1]
        use = inside or [min(self.samples, key=lambda ts: abs(ts[0] - (t0 + t1) / 2))[1]]

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        sm = sorted(x for x in (num(s[1]) for s in use) if x is not None)
        mx = [num(s[2]) for s in use if num(s[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in use for i in range(4) if s[5 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(use), "samples_in_timed_region": len(inside),
                "power_w_max": max((num(s[3]) or 0.0) for s in use)}


# ----------------------------------------------------------------------------- multi-rank host logic
def _dist():
    from paper_2401_06197_b200.sharding import dist_env
    return dist_env()


def _shard(batch, ws, rank, shard):
    from paper_2401_06197_b200.sharding import shard_images
    return shard_images(batch, ws, rank) if shard else list(range(batch))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(nproc: int, argv) -> int:
    """`--gpus N` outside torchrun: re-run this script under torch.distributed.run with N
    ranks on this node (rendezvous on 127.0.0.1), NCCL init logging on; returns the exit
    status of the launcher (rank 0 prints the JSON line)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def max_over_ranks(v: float, ws: int, dist, device) -> float:
    """The slowest rank's value (step times are reported as the max over ranks)."""
    if ws <= 1:
        return v
    import torch
    t = torch.tensor([v], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cross_rank_check(first_image: int, outputs, recompute, ws: int, rank: int, dist, device):
    """N > 1: gather every rank's first-image outputs (a list of tensors, one per
    (stage, tensor)) to rank 0, which recomputes those images alone with
    recompute(image, index) and requires bit-identical results (forward and
    grad_offset_mask do not depend on the batch partition, R14).
    Returns {"cross_rank_bitexact": bool, "ranks": ws} on rank 0, None elsewhere."""
    import torch
    first = torch.tensor([first_image], device=device, dtype=torch.int64)
    firsts = [torch.zeros_like(first) for _ in range(ws)]
    dist.all_gather(firsts, first)
    ok = True
    for idx, mine in enumerate(outputs):
        mine = mine.contiguous()
        got = [torch.empty_like(mine) for _ in range(ws)] if rank == 0 else None
        dist.gather(mine, got, dst=0)
        if rank != 0:
            continue
        for r in range(ws):
            ref = recompute(int(firsts[r].item()), idx)
            ok = ok and bool(torch.equal(ref.to(got[r].device), got[r]))
    return {"cross_rank_bitexact": ok, "ranks": ws} if rank == 0 else None


# ----------------------------------------------------------------------------- bytes
def _alg_bytes(x, om, backward, w=None):
    """Algorithmic bytes of one call: forward x + om + y; backward
    x + om + gy (reads) + gx + gom (writes).  y/gy/gx are x-sized, gom is om-sized.
    Fused module (w given): x + W + y -- the offset_mask is never in memory."""
    bx = x.numel() * x.element_size()
    if w is not None:
        return 2 * bx + w.numel() * w.element_size()
    bo = om.numel() * om.element_size()
    return (3 * bx + 2 * bo) if backward else (2 * bx + bo)


def _call_bytes(cfg, st, kind):
    """Algorithmic bytes of one call of a stage: _alg_bytes for the operator / lightweight
    module; for the full module (R22) every tensor each GEMM / kernel must read or write
    once (A = activation bytes [N,H,W,C], O = offset_mask bytes [N,H,W,S], Wt = weights):
      fwd          v = lin(x), a = core(x, v), y = lin(a):      7A + Wt
      fwd_unfused  + om = lin(x) written and read back:         6A + 2O + Wt
      bwd          ga, dW_out, om recompute, DCNv4 bwd, gx, dW_in, dW_om:  13A + 5O + 2 Wt"""
    if cfg.get("module") != "full":
        return _alg_bytes(st["x"], st["om"], kind == "bwd", st.get("w"))
    A = st["x"].numel() * st["x"].element_size()
    S = -(-27 * st["G"] // 8) * 8
    O = A // st["x"].shape[-1] * S
    Wt = sum(v.numel() * v.element_size() for v in st["params"].values())
    return {"fwd": 7 * A + Wt, "fwd_unfused": 6 * A + 2 * O + Wt, "bwd": 13 * A + 5 * O + 2 * Wt}[kind]


def _traffic(workload, kind):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return int(t[workload][kind])
    except Exception:
        return None


# ----------------------------------------------------------------------------- oracle arm
def oracle_inputs(cfg, images):
    """The sample's inputs (same seeded generator as the GPU arm), as fp64 arrays."""
    import oracle
    import synth
    oracle.build()
    data = []
    for (H, W, G, D) in cfg["stages"]:
        g = oracle.Geometry(N=len(images), H=H, W=W, G=G, D=D)
        x, om, gy = synth.make_case(len(images), H, W, G, D, H, W, K, 27 * G, cfg["dtype"],
                                    images=images)
        if cfg.get("module") == "full":
            prm = {k: oracle._f64(v) for k, v in synth.make_module_params(G * D, G, K, cfg["dtype"]).items()}
            data.append((g, oracle._f64(x), prm, oracle._f64(gy)))
            continue
        if cfg.get("module"):  # om comes from the linear: carry (weight, bias) instead
            w, b = synth.make_linear(G * D, G, K, cfg["dtype"])
            om = (oracle._f64(w), oracle._f64(b))
            data.append((g, oracle._f64(x), om, None))
            continue
        data.append((g, oracle._f64(x), oracle._f64(om), oracle._f64(gy)))
    return data


def oracle_sample(cfg, data):
    """Time the fp64 oracle (as it stands) over `data`: every stage, forward (+ backward).
    Returns seconds."""
    import oracle
    t0 = time.perf_counter()
    for g, x, om, gy in data:
        if cfg.get("module") == "full":
            if cfg["backward"]:
                oracle.module_full_backward(g, x, om, gy, cfg["dtype"])  # includes the forward
            else:
                oracle.module_full_forward(g, x, om, cfg["dtype"])
            continue
        if cfg.get("module"):
            oracle.module_forward(g, x, om[0], om[1], cfg["dtype"])
            continue
        oracle.forward(g, x, om)
        if cfg["backward"]:
            oracle.backward(g, x, om, gy)
    return time.perf_counter() - t0


def cpu_baseline(cfg, target_s=12.0):
    t1 = oracle_sample(cfg, oracle_inputs(cfg, [0, 1]))
    n = int(max(2, min(cfg["batch"], round(2 * target_s / max(t1, 1e-3)))))
    t = oracle_sample(cfg, oracle_inputs(cfg, list(range(n)))) if n > 2 else t1
    return {"value": n / t, "unit": "imgs/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
            "kind": "oracle",
            "sample": f"{n} images of workload {cfg['name']} (all stages, "
                      f"{'fwd+bwd' if cfg['backward'] else 'fwd'}), fp64 C oracle, "
                      f"OpenMP over (image, group), {t:.1f} s"}


def run_reference(args, cfg):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    steps = args.steps or 2
    budget = 60.0
    t2 = oracle_sample(cfg, oracle_inputs(cfg, [0, 1])) / 2
    n = int(max(1, min(cfg["batch"], budget / max(1, steps + args.warmup) / max(t2, 1e-3))))
    data = oracle_inputs(cfg, list(range(n)))
    for _ in range(args.warmup):
        oracle_sample(cfg, data)
    times = [oracle_sample(cfg, data) for _ in range(steps)]
    tot = sum(times)
    value = n * steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "imgs/s", "n_gpus": ws,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / steps,
        "higher_is_better": True, "scaling": "strong" if cfg["shard"] else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "desc": cfg["desc"], "global_batch": cfg["batch"],
                   "images_per_step_sample": n},
        "cpu_baseline": {"value": value, "unit": "imgs/s", "kind": "oracle",
                         "cores": int(os.environ["OMP_NUM_THREADS"]),
                         "sample": f"{n} images per step of workload {cfg['name']} "
                                   f"(all stages, {'fwd+bwd' if cfg['backward'] else 'fwd'})"},
        "e2e": {"value": value, "unit": "imgs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
class Ctx:
    """Per-process run context (device, ranks, streams, clock sampler)."""

    def __init__(self, torch, dist, pkg, dev, ws, rank):
        self.torch, self.dist, self.pkg, self.dev, self.ws, self.rank = torch, dist, pkg, dev, ws, rank
        self.stream = torch.cuda.Stream(device=dev)
        self.l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
        uuid = None
        try:
            uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
        except Exception:
            pass
        self.sampler = ClockSampler(uuid)


def _make_stages(cfg, ctx, images, offsets, deterministic):
    import synth
    torch, pkg, dev = ctx.torch, ctx.pkg, ctx.dev
    tdt = synth.DTYPES[cfg["dtype"]]
    stages = []
    for (H, W, G, D) in cfg["stages"]:
        x, om, gy = synth.make_case(len(images), H, W, G, D, H, W, K, 27 * G, cfg["dtype"],
                                    images=images, offsets=offsets, with_gy=cfg["backward"])
        st = dict(H=H, W=W, G=G, D=D, x_cpu=x, om_cpu=om, gy_cpu=gy, x=x.to(dev), om=om.to(dev),
                  gy=gy.to(dev) if gy is not None else None)
        if cfg.get("module") == "full":
            prm = synth.make_module_params(G * D, G, K, cfg["dtype"])
            st.update(params_cpu=prm, params={k: v.to(dev) for k, v in prm.items()})
        elif cfg.get("module"):
            w, b = synth.make_linear(G * D, G, K, cfg["dtype"])
            st.update(w_cpu=w, b_cpu=b, w=w.to(dev), b=b.to(dev))
        st["y"] = torch.empty_like(st["x"])
        if cfg["backward"] and cfg.get("module") != "full":
            st["gx"] = torch.empty_like(st["x"])
            st["gom"] = torch.empty_like(st["om"])
            need = pkg.workspace_bytes(pkg.make_params(len(images), H, W, G, D,
                                                       deterministic=deterministic), tdt)
            st["ws"] = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
        stages.append(st)
    return stages


def _calls(cfg, st, pkg, softmax, deterministic):
    if cfg.get("module") == "full":
        M = pkg.module

        def fwd():
            st["y"], st["saved"] = M.full_forward(st["x"], st["params"], st["G"], softmax=softmax)

        def fwd_unfused():  # the multi-call path: 4 launches, om through memory
            p = st["params"]
            v = M.linear(st["x"], p["w_in"], p["b_in"])
            om = M.offset_mask_linear(st["x"], p["w_om"], p["b_om"], st["G"])
            a = pkg.forward(v, om, group=st["G"], softmax=softmax)
            st["y_unfused"] = M.linear(a, p["w_out"], p["b_out"])

        out = [("fwd", fwd), ("fwd_unfused", fwd_unfused)]
        if cfg["backward"]:
            out.append(("bwd", lambda: st.__setitem__("grads", M.full_backward(
                st["x"], st["params"], st["G"], st["gy"], st["saved"], softmax=softmax))))
        return out
    if cfg.get("module"):
        return [("fwd", lambda: pkg.module.forward_fused(st["x"], st["w"], st["b"], st["G"],
                                                         softmax=softmax, out=st["y"]))]
    out = [("fwd", lambda: pkg.forward(st["x"], st["om"], group=st["G"], softmax=softmax,
                                       out=st["y"]))]
    if cfg["backward"]:
        out.append(("bwd", lambda: pkg.backward(
            st["x"], st["om"], st["gy"], group=st["G"], softmax=softmax, grad_input=st["gx"],
            grad_offset_mask=st["gom"], workspace=st["ws"], deterministic=deterministic)))
    return out


def measure(cfg, ctx, images, steps, warmup, offsets="u2", softmax=False, deterministic=False,
            verify=True):
    """Time `steps` steps of workload `cfg` on this rank's `images`; returns a dict with the
    max-over-ranks step time, the per-stage table, the dominant kernel's roofline, the
    clocks sampled during the timed region and the parity record."""
    torch, pkg, dev, stream, ws, rank = ctx.torch, ctx.pkg, ctx.dev, ctx.stream, ctx.ws, ctx.rank
    stages = _make_stages(cfg, ctx, images, offsets, deterministic)
    if cfg.get("grouped"):  # every stage in one dcnv4_forward_grouped launch
        def grouped():
            pkg.forward_grouped([s["x"] for s in stages], [s["om"] for s in stages], [s["G"] for s in stages],
                                softmax=softmax, outs=[s["y"] for s in stages])
        step_calls = [(0, "fwd", grouped)]
    else:
        step_calls = [(si, kind, fn) for si, st in enumerate(stages)
                      for kind, fn in _calls(cfg, st, pkg, softmax, deterministic)]
    work_set = sum(_call_bytes(cfg, s, "fwd") + (_call_bytes(cfg, s, "bwd") if cfg["backward"] else 0)
                   for s in stages)
    flush_bytes = 0
    if work_set < 2 * ctx.l2_bytes:
        # the step's data could stay in L2 between steps: write a 2xL2 buffer after every
        # step (timed by its own events and excluded from the step time)
        flush_bytes = 2 * ctx.l2_bytes
        l2buf = torch.empty(flush_bytes, dtype=torch.uint8, device=dev)
        step_calls.append((-1, "flush", lambda: l2buf.fill_(1)))

    # one eager step (outputs kept for verification outside the timed region)
    with torch.cuda.stream(stream):
        for _, _, fn in step_calls:
            fn()
    stream.synchronize()
    parity = None
    if verify and ws == 1:
        parity = _verify(cfg, stages, images, softmax=softmax)
    elif verify and ws > 1:
        parity = _cross_rank(cfg, stages, images, ctx, softmax)

    # warm-up (eager), then capture up to GRAPH_STEPS steps with event nodes between calls
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            for _, _, fn in step_calls:
                fn()
    stream.synchronize()
    if steps is None:  # auto: a timed region of >= MIN_TIMED_S, in whole graphs
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            for _, _, fn in step_calls:
                fn()
            b.record(stream)
        stream.synchronize()
        est = max(a.elapsed_time(b), 1e-3)
        steps = max(20, math.ceil(MIN_TIMED_S * 1e3 / est))
        if steps > GRAPH_STEPS:
            steps = math.ceil(steps / GRAPH_STEPS) * GRAPH_STEPS
    gsteps = steps if steps <= GRAPH_STEPS else GRAPH_STEPS
    if steps % gsteps:
        raise ValueError(f"--steps {steps} > {GRAPH_STEPS} must be a multiple of {GRAPH_STEPS}")
    replays = steps // gsteps
    n_calls = len(step_calls)
    evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(gsteps * n_calls + 1)]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        evs[0].record(stream)
        e = 1
        for _ in range(gsteps):
            for _, _, fn in step_calls:
                fn()
                evs[e].record(stream)
                e += 1
    graph.replay()  # one untimed replay (graph upload, warm)
    stream.synchronize()

    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    time.sleep(0.2)
    if ws > 1:
        ctx.dist.barrier()
    torch.cuda.synchronize(dev)
    t_wall0 = time.time()
    with torch.cuda.stream(stream):
        t_start.record(stream)
        for _ in range(replays):
            graph.replay()
        t_end.record(stream)
    torch.cuda.synchronize(dev)
    t_wall1 = time.time()
    if ws > 1:
        ctx.dist.barrier()
    time.sleep(0.1)
    clocks = ctx.sampler.summary(t_wall0, t_wall1)

    total_ms = t_start.elapsed_time(t_end)
    durs = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)]  # last replay
    per_call = {}
    flush_ms = 0.0
    for i, d in enumerate(durs):
        si, kind, _ = step_calls[i % n_calls]
        if kind in ("flush", "fwd_unfused"):  # timed separately, not part of the step
            flush_ms += d
            if kind == "flush":
                continue
        per_call.setdefault((si, kind), []).append(d)
    flush_per_step = flush_ms / gsteps
    ms_step = max_over_ranks((total_ms - flush_per_step * steps) / steps, ws, ctx.dist, dev)

    peak, peak_src = _peaks()
    table = []
    kind_bytes, kind_ms = {}, {}
    paper = PAPER_A100_MS.get(cfg.get("paper"), {}).get(cfg["dtype"])
    for si, st in enumerate(stages):
        row = {"shape": shape_name(st["H"], st["W"], st["G"], st["D"]), "images": len(images)}
        if cfg.get("grouped") and si == 0:
            row["shape"] = "all stages, one grouped launch: " + ", ".join(
                shape_name(q["H"], q["W"], q["G"], q["D"]) for q in stages)
        for kind in ("fwd", "bwd", "fwd_unfused"):
            if (si, kind) not in per_call:
                continue
            ms = sum(per_call[(si, kind)]) / len(per_call[(si, kind)])
            b = (sum(_call_bytes(cfg, q, kind) for q in stages) if cfg.get("grouped")
                 else _call_bytes(cfg, st, kind))
            gbs = b / (ms * 1e-3) / 1e9
            srt = sorted(per_call[(si, kind)])
            pick = lambda q: srt[min(len(srt) - 1, int(q * (len(srt) - 1) + 0.5))]  # noqa: E731
            row[f"{kind}_us"] = round(ms * 1e3, 2)
            row[f"{kind}_us_p10_p50_p90"] = [round(pick(q) * 1e3, 2) for q in (0.1, 0.5, 0.9)]
            row[f"{kind}_GBs"] = round(gbs, 1)
            row[f"{kind}_frac"] = round(gbs / peak, 4)
            if kind == "fwd_unfused":  # reported beside the fused path, not part of the step
                continue
            kind_bytes[kind] = kind_bytes.get(kind, 0) + b
            kind_ms[kind] = kind_ms.get(kind, 0.0) + ms
        if paper and si < len(paper):
            row["paper_a100_fwd_us"] = round(paper[si] * 1e3, 1)
        # checksum: fp64 sums of the outputs of the last step
        row["checksum"] = {"y": float(st["y"].double().sum())}
        if cfg.get("module") == "full":
            if cfg["backward"]:
                row["checksum"].update({f"grad_{k}": float(v.double().sum()) for k, v in st["grads"].items()})
        elif cfg["backward"]:
            row["checksum"]["grad_offset_mask"] = float(st["gom"].double().sum())
            row["checksum"]["grad_input"] = float(st["gx"].double().sum())
        table.append(row)
    dom = max(kind_ms, key=kind_ms.get)
    launches_dom = 1 if cfg.get("grouped") else len(stages)
    achieved = kind_bytes[dom] / (kind_ms[dom] * 1e-3) / 1e9
    share = kind_ms[dom] / sum(kind_ms.values())
    if cfg.get("module") == "full":
        kname = ("full-module backward: tcgen05 GEMMs + offset/mask linear + memset + bwd33_kernel"
                 if dom == "bwd" else "full-module forward: tcgen05 linear + module_fwd_kernel + tcgen05 linear")
    else:
        kname = "memset + bwd33_kernel" if dom == "bwd" else (
            "module_fwd_kernel: tcgen05 linear + aggregation" if cfg.get("module") else
            "fwd33_group_kernel (all stages)" if cfg.get("grouped") else "fwd33_kernel")
    roofline = {"bound": "hbm", "kernel": f"dcnv4 {dom} ({kname}), {launches_dom} launches per step",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_src,
                "traffic": _traffic(cfg["name"], dom), "share_of_step": round(share, 4),
                "alg_bytes_per_launch": int(kind_bytes[dom] / launches_dom)}
    l2 = (f"step working set {work_set / 1e6:.1f} MB < 2x L2 ({2 * ctx.l2_bytes >> 20} MB): "
          f"a {flush_bytes >> 20} MB buffer written after every step, timed separately and "
          f"excluded" if flush_bytes else
          f"inputs larger than L2: step working set {work_set / 1e9:.2f} GB vs "
          f"{ctx.l2_bytes >> 20} MB L2; no flush")
    return {"stages": stages, "ms_step": ms_step, "steps": steps, "table": table,
            "roofline": roofline, "clocks": clocks, "parity": parity, "l2": l2,
            "wall_s": round(t_wall1 - t_wall0, 4), "replays": replays}


def _verify(cfg, stages, images, softmax=False):
    """Oracle check of the shard's first image on every stage (outside the timed region)."""
    import oracle
    out = {}
    tol = 1e-5 if cfg["dtype"] == "f32" else 1e-2
    for st in stages:
        g = oracle.Geometry(N=1, H=st["H"], W=st["W"], G=st["G"], D=st["D"], softmax=softmax)
        if cfg.get("module") == "full":  # forward of the first image (weight grads sum the batch)
            fw = oracle.module_full_forward(g, st["x_cpu"][:1], st["params_cpu"], cfg["dtype"], with_abs=True)
            out[shape_name(st["H"], st["W"], st["G"], st["D"])] = {
                "y": float(f"{oracle.abs_scaled_error(st['y'][:1].cpu(), fw['y'], fw['y_abs']):.3e}")}
            continue
        if cfg.get("module"):
            y_ref, y_abs, _ = oracle.module_forward(g, st["x_cpu"][:1], st["w_cpu"], st["b_cpu"],
                                                    cfg["dtype"], with_abs=True)
        else:
            y_ref, y_abs = oracle.forward(g, st["x_cpu"][:1], st["om_cpu"][:1], with_abs=True)
        errs = {"y": oracle.abs_scaled_error(st["y"][:1].cpu(), y_ref, y_abs)}
        if cfg["backward"] and not cfg.get("module"):
            gx_ref, gom_ref, gxa, goma = oracle.backward(g, st["x_cpu"][:1], st["om_cpu"][:1],
                                                         st["gy_cpu"][:1], with_abs=True)
            errs["grad_input"] = oracle.abs_scaled_error(st["gx"][:1].cpu(), gx_ref, gxa)
            errs["grad_offset_mask"] = oracle.abs_scaled_error(st["gom"][:1].cpu(), gom_ref, goma)
        out[shape_name(st["H"], st["W"], st["G"], st["D"])] = {k: float(f"{v:.3e}") for k, v in errs.items()}
    worst = max(v for e in out.values() for v in e.values())
    return {"image": images[0], "max_abs_scaled_error": worst, "tol": tol,
            "pass": bool(worst <= tol), "per_stage": out}


def _cross_rank(cfg, stages, images, ctx, softmax):
    import synth
    pkg = ctx.pkg
    keys = ("y", "gom") if cfg["backward"] else ("y",)
    outputs = [st[k][:1] for st in stages for k in keys]

    def recompute(n, idx):
        st, key = stages[idx // len(keys)], keys[idx % len(keys)]
        x, om, gy = synth.make_case(1, st["H"], st["W"], st["G"], st["D"], st["H"], st["W"], K,
                                    27 * st["G"], cfg["dtype"], images=[n])
        x, om = x.to(ctx.dev), om.to(ctx.dev)
        if key == "y" and cfg.get("module"):
            return pkg.module.forward_fused(x, st["w"], st["b"], st["G"], softmax=softmax)
        if key == "y":
            return pkg.forward(x, om, group=st["G"], softmax=softmax)
        return pkg.backward(x, om, gy.to(ctx.dev), group=st["G"], softmax=softmax)[1]
    return cross_rank_check(images[0], outputs, recompute, ctx.ws, ctx.rank, ctx.dist, ctx.dev)


def _e2e(args, cfg, stages, ctx):
    """Same metric through the public API with pinned host buffers: every step copies the
    step's inputs host->device and its results device->host inside the timed region."""
    torch, pkg, dev, ws = ctx.torch, ctx.pkg, ctx.dev, ctx.ws
    host = []
    h2d = d2h = 0
    for st in stages:
        h = {"x": st["x_cpu"].pin_memory(), "om": st["om_cpu"].pin_memory(),
             "y": torch.empty_like(st["x_cpu"]).pin_memory()}
        # module: the offset_mask is computed on the device from x (weights stay resident)
        h2d += sum(h[k].numel() * h[k].element_size()
                   for k in (("x",) if cfg.get("module") else ("x", "om")))
        d2h += h["y"].numel() * h["y"].element_size()
        if cfg["backward"]:
            h["gy"] = st["gy_cpu"].pin_memory()
            h["gx"] = torch.empty_like(st["x_cpu"]).pin_memory()
            h2d += h["gy"].numel() * h["gy"].element_size()
            if cfg.get("module") == "full":  # grad_input and every weight / bias gradient
                h["gw"] = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in st["params"].items()}
                d2h += h["gx"].numel() * h["gx"].element_size() + sum(
                    v.numel() * v.element_size() for v in h["gw"].values())
            else:
                h["gom"] = torch.empty_like(st["om_cpu"]).pin_memory()
                d2h += sum(h[k].numel() * h[k].element_size() for k in ("gx", "gom"))
        host.append(h)

    # chunked over images on three streams (paper_2401_06197_b200/pipeline.py): the H2D
    # copies of chunk c+1, the library calls of chunk c and the D2H copies of chunk c-1
    # overlap; every byte of every step still crosses the host link inside the timed region
    from paper_2401_06197_b200.pipeline import HostPipeline
    nimg = len(stages[0]["x"])
    nch = max(1, min(args.e2e_chunks, nimg))
    if cfg.get("module") == "full" and cfg["backward"]:
        nch = 1  # the weight gradients sum over the whole batch: one chunk
    bounds = [(c * nimg // nch, (c + 1) * nimg // nch) for c in range(nch)]
    pipe = HostPipeline(dev, nch)

    def copy_in(c):
        lo, hi = bounds[c]
        for st, h in zip(stages, host):
            st["x"][lo:hi].copy_(h["x"][lo:hi], non_blocking=True)
            if not cfg.get("module"):
                st["om"][lo:hi].copy_(h["om"][lo:hi], non_blocking=True)
            if cfg["backward"]:
                st["gy"][lo:hi].copy_(h["gy"][lo:hi], non_blocking=True)

    def compute(c):
        lo, hi = bounds[c]
        for st in stages:
            if cfg.get("module") == "full":
                M = pkg.module
                y, saved = M.full_forward(st["x"][lo:hi], st["params"], st["G"], softmax=args.softmax)
                st["y"][lo:hi].copy_(y)
                if cfg["backward"]:
                    st["grads"] = M.full_backward(st["x"][lo:hi], st["params"], st["G"], st["gy"][lo:hi],
                                                  saved, softmax=args.softmax)
                continue
            if cfg.get("module"):
                pkg.module.forward_fused(st["x"][lo:hi], st["w"], st["b"], st["G"],
                                         softmax=args.softmax, out=st["y"][lo:hi])
                continue
            pkg.forward(st["x"][lo:hi], st["om"][lo:hi], group=st["G"], softmax=args.softmax,
                        out=st["y"][lo:hi])
            if cfg["backward"]:
                pkg.backward(st["x"][lo:hi], st["om"][lo:hi], st["gy"][lo:hi], group=st["G"],
                             softmax=args.softmax, grad_input=st["gx"][lo:hi],
                             grad_offset_mask=st["gom"][lo:hi], workspace=st["ws"],
                             deterministic=args.deterministic)

    def copy_out(c):
        lo, hi = bounds[c]
        for st, h in zip(stages, host):
            h["y"][lo:hi].copy_(st["y"][lo:hi], non_blocking=True)
            if cfg["backward"] and cfg.get("module") == "full":
                h["gx"][lo:hi].copy_(st["grads"]["x"], non_blocking=True)
                for k, v in h["gw"].items():
                    v.copy_(st["grads"][k], non_blocking=True)
            elif cfg["backward"]:
                h["gx"][lo:hi].copy_(st["gx"][lo:hi], non_blocking=True)
                h["gom"][lo:hi].copy_(st["gom"][lo:hi], non_blocking=True)

    pipe.run(copy_in, compute, copy_out)  # warm-up pass
    torch.cuda.synchronize(dev)
    if ws > 1:
        ctx.dist.barrier()
    torch.cuda.synchronize(dev)
    evs = [pipe.run(copy_in, compute, copy_out) for _ in range(args.e2e_steps)]
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(evs[0][0].elapsed_time(evs[-1][1]) / args.e2e_steps, ws, ctx.dist, dev)
    n_total = cfg["batch"] if cfg["shard"] else ws * len(stages[0]["x"])
    return {"value": round(n_total / (ms * 1e-3), 2), "unit": "imgs/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(ms, 3), "steps": args.e2e_steps, "chunks": nch,
            "overlap": "H2D / kernels / D2H on three streams, chunked by image"}


def _extras(args, ctx):
    """Forward sweeps of the default run: per-stage µs / GB/s / fraction of
    HBM, the paper's A100 rows beside the D=32 sets, first-image oracle parity, clocks."""
    out = []
    for name, batch in EXTRAS:
        cfg = dict(WORKLOADS[name], name=name)
        if batch:
            cfg["batch"] = batch
        try:
            r = measure(cfg, ctx, list(range(cfg["batch"])), None, args.warmup)
        except Exception as e:  # a sweep must not sink the headline line
            out.append({"workload": name, "batch": cfg["batch"], "error": repr(e)[:300]})
            continue
        tot_b = sum(_alg_bytes(s["x"], s["om"], cfg["backward"]) for s in r["stages"])
        out.append({
            "workload": name, "desc": cfg["desc"], "dtype": cfg["dtype"], "batch": cfg["batch"],
            "imgs_per_s": round(cfg["batch"] / (r["ms_step"] * 1e-3), 1),
            "us_per_step": round(r["ms_step"] * 1e3, 2), "steps": r["steps"],
            "aggregate_GBs": round(tot_b / (r["ms_step"] * 1e-3) / 1e9, 1),
            "aggregate_frac": round(tot_b / (r["ms_step"] * 1e-3) / 1e9 / _peaks()[0], 4),
            "stages": [{k: v for k, v in row.items() if k != "checksum"} for row in r["table"]],
            "roofline_frac_dominant": r["roofline"]["frac"], "l2": r["l2"],
            "clocks": r["clocks"], "parity": r["parity"]})
        for st in r["stages"]:
            st.clear()
        ctx.torch.cuda.empty_cache()
    return out


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 50 for c4, else a >= 0.4 s timed region)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--global-batch", type=int, default=0)
    ap.add_argument("--offsets", default="u2", choices=["u2", "zero", "u8", "smooth"])
    ap.add_argument("--softmax", action="store_true",
                    help="DCNv3 mode (softmax over K, NEXT-1) instead of DCNv4")
    ap.add_argument("--deterministic", action="store_true",
                    help="bit-reproducible grad_input (int64 fixed point, NEXT-4)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=8,
                    help="image chunks of the host-streaming e2e pipeline (1 = no overlap)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the forward sweeps")
    ap.add_argument("--out", default="", help="also append the JSON line to this file")
    args = ap.parse_args(argv)
    ws, rank, local = _dist()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus, argv)
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using the launcher's {ws} ranks",
              file=sys.stderr)
    cfg = dict(WORKLOADS[args.workload], name=args.workload)
    if args.global_batch:
        cfg["batch"] = args.global_batch
    if args.steps is None and args.workload == "c4":
        args.steps = 50
    if args.warmup < 3:
        args.warmup = 3  # contract: >= 3 untimed warm-up steps
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2401_06197_b200 as pkg

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = Ctx(torch, dist, pkg, dev, ws, rank)
    images = _shard(cfg["batch"], ws, rank, cfg["shard"])
    n_img = len(images)
    r = measure(cfg, ctx, images, args.steps, args.warmup, args.offsets, bool(args.softmax),
                args.deterministic, verify=not args.no_verify and not (ws == 1 and args.no_cpu_baseline))
    ms_step = r["ms_step"]
    value = cfg["batch"] / (ms_step * 1e-3) if cfg["shard"] else ws * n_img / (ms_step * 1e-3)
    stages = r["stages"]

    e2e = _e2e(args, cfg, stages, ctx)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)
    extras = None
    if ws == 1 and not args.no_extras and args.workload == "c4":
        for st in stages:
            st.clear()
        torch.cuda.empty_cache()
        extras = _extras(args, ctx)
    ctx.sampler.stop()

    n_ours = (2 if cfg["backward"] else 1) * (1 if cfg.get("grouped") else len(stages))
    if cfg["backward"] and args.deterministic:
        n_ours += 2 * len(stages)  # per-image maxima + int64 -> T conversion
    elif cfg["backward"] and cfg["dtype"] != "f32":
        n_ours += len(stages)  # fp32 -> half grad_input conversion
    detail = (f"per step: {len(stages)} "
              + ("module_fwd_kernel" if cfg.get("module") else "fwd33_kernel")
              + (f" + {len(stages)} bwd33_kernel + {len(stages)} accumulator "
                 f"zero-fill (cudaMemsetAsync)" if cfg["backward"] else "")
              + (f" + {len(stages)} det_scale_kernel + {len(stages)} det_convert_kernel"
                 if cfg["backward"] and args.deterministic else
                 f" + {len(stages)} convert_kernel" if cfg["backward"] and cfg["dtype"] != "f32"
                 else ""))
    if cfg.get("module") == "full":
        # per stage: forward 3 (gemm, module_fwd, gemm) + the unfused comparison path 4
        # (gemm, om_linear, fwd33, gemm; its time is excluded from the step); backward 17
        # (3 x grad_weight: gemm + colsum + 2 conversions; 2 grad_input gemms; om_linear;
        # bwd33 + convert)
        n_ours = len(stages) * (3 + 4 + (17 if cfg["backward"] else 0))
        detail = (f"per stage and step: forward gemm_kernel + module_fwd_kernel + gemm_kernel; unfused "
                  f"comparison gemm_kernel + om_linear_kernel + fwd33_kernel + gemm_kernel"
                  + ("; backward 3 x (gemm_kernel + colsum_kernel + 2 f32_to_t_kernel) + 2 gemm_kernel + "
                     "om_linear_kernel + bwd33_kernel + convert_kernel (+ 4 cudaMemsetAsync)"
                     if cfg["backward"] else ""))
    Ds = sorted({d for *_, d in cfg["stages"]})
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "imgs/s", "n_gpus": ws,
        "steps": r["steps"], "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "strong" if cfg["shard"] else "weak",
        "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
        "config": {"workload": cfg["name"], "desc": cfg["desc"], "global_batch": cfg["batch"],
                   "per_gpu_batch": n_img, "stages": [shape_name(*s) for s in cfg["stages"]],
                   "D": Ds[0] if len(Ds) == 1 else Ds, "kernel": "3x3 s1 p1 d1",
                   "offset_scale": 1.0, "offsets": args.offsets,
                   "operator": "DCNv3 (softmax over K)" if args.softmax else "DCNv4",
                   "grad_input": ("deterministic int64 fixed point" if args.deterministic
                                  else "fp32 atomics") if cfg["backward"] else None,
                   "parallelism": f"batch-sharded dp{ws}" if cfg["shard"] else f"replicas x{ws}",
                   "l2": r["l2"]},
        "roofline": r["roofline"],
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": n_ours * r["steps"],
        "gpu_launch_detail": detail,
        "clocks": r["clocks"],
        "stages": r["table"],
        "parity": r["parity"],
        "wall_s_timed_region": r["wall_s"],
        "forward_sweeps": extras,
    }
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
