"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws random numbers of the
shapes, ranges and structure of the paper's workloads (DESIGN.md "Input recipe",
SURVEY.md 8(d).1).  Both the oracle side and the CUDA side receive the same tensors.

Recipe (per image n, global index ``n`` so 1/2/4/8-rank shards see identical images):
  seed(tensor_id, n) = 20240111 + 1000 * tensor_id + n   (tensor_id: x=0, om=1, gy=2)
  x  ~ U(-1, 1)                      input feature map, NHWC  [N, H, W, G*D]
  dx, dy ~ U(-2, 2) i.i.d.           offsets (SPEC S:133 seeded case), in offset_mask
  m  ~ U(-1, 1)                      unnormalised modulation ("unbounded")
  padding channels of offset_mask (S > 3GK) ~ U(-1, 1) (must be ignored)
  gy ~ U(-1, 1)                      upstream gradient, NHWC [N, Ho, Wo, G*D]
Values are drawn in fp32 with torch's CPU generator and then cast (RN-even) to the
storage dtype; the oracle is fed the same quantised values.
Offset variants: "u2" (default), "zero", "u8" (weak locality), "smooth" (coarse 8x8
U(-2,2) field upsampled bilinearly, mimicking learned offsets).
"""
from __future__ import annotations

import torch

SEED_BASE = 20240111
TENSOR_X, TENSOR_OM, TENSOR_GY = 0, 1, 2

DTYPES = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}


def seed_of(tensor_id: int, image: int) -> int:
    return SEED_BASE + 1000 * tensor_id + image


def _uniform(shape, seed, lo, hi):
    g = torch.Generator().manual_seed(seed)
    return torch.rand(shape, generator=g, dtype=torch.float32) * (hi - lo) + lo


def image_x(H, W, C, image):
    return _uniform((H, W, C), seed_of(TENSOR_X, image), -1.0, 1.0)


def image_gy(Ho, Wo, C, image):
    return _uniform((Ho, Wo, C), seed_of(TENSOR_GY, image), -1.0, 1.0)


def image_om(Ho, Wo, G, K, S, image, offsets="u2"):
    """One image's fused offset_mask row block [Ho, Wo, S] (layout: DESIGN.md R3)."""
    g = torch.Generator().manual_seed(seed_of(TENSOR_OM, image))
    om = torch.rand((Ho, Wo, S), generator=g, dtype=torch.float32) * 2.0 - 1.0  # m, pad
    off = torch.rand((Ho, Wo, G, 2 * K), generator=g, dtype=torch.float32)
    if offsets == "u2":
        off = off * 4.0 - 2.0
    elif offsets == "u8":
        off = off * 16.0 - 8.0
    elif offsets == "zero":
        off = torch.zeros_like(off)
    elif offsets == "smooth":
        coarse = torch.rand((1, G * 2 * K, 8, 8), generator=g) * 4.0 - 2.0
        up = torch.nn.functional.interpolate(coarse, size=(Ho, Wo), mode="bilinear",
                                             align_corners=True)
        off = up[0].permute(1, 2, 0).reshape(Ho, Wo, G, 2 * K)
    else:
        raise ValueError(f"unknown offset distribution {offsets!r}")
    for grp in range(G):
        om[:, :, grp * 3 * K: grp * 3 * K + 2 * K] = off[:, :, grp]
    return om


def make_case(N, H, W, G, D, Ho, Wo, K, S, dtype="f32", images=None, offsets="u2",
              with_gy=True):
    """CPU tensors (x, om, gy) for images ``images`` (default range(N)) in ``dtype``."""
    images = list(range(N)) if images is None else list(images)
    C = G * D
    dt = DTYPES[dtype]
    x = torch.stack([image_x(H, W, C, n) for n in images]).to(dt) if images else \
        torch.empty((0, H, W, C), dtype=dt)
    om = torch.stack([image_om(Ho, Wo, G, K, S, n, offsets) for n in images]).to(dt) \
        if images else torch.empty((0, Ho, Wo, S), dtype=dt)
    gy = None
    if with_gy:
        gy = torch.stack([image_gy(Ho, Wo, C, n) for n in images]).to(dt) if images else \
            torch.empty((0, Ho, Wo, C), dtype=dt)
    return x, om, gy


# ---------------------------------------------------------------------------------------
# Multi-scale deformable attention inputs (NEXT-3, R20).
#   value ~ U(-1, 1)                    [N, S, M, D], S = sum_l H_l*W_l
#   loc   ~ U(-0.1, 1.1) (x, y)         [N, Lq, M, L, P, 2]: normalised sampling points,
#                                       a margin outside [0, 1] exercises zero padding
#   attn  ~ U(0, 2/(L*P))               [N, Lq, M, L, P]: positive weights summing to ~1
#                                       per (query, head), like the caller's softmax
#   gout  ~ U(-1, 1)                    [N, Lq, M, D]
TENSOR_VALUE, TENSOR_LOC, TENSOR_ATTN, TENSOR_GOUT = 10, 11, 12, 13


def make_msda_case(N, Lq, M, D, P, shapes, dtype="f32", images=None, loc_range=(-0.1, 1.1),
                   with_gout=True):
    """CPU tensors (value, loc, attn, gout) for images ``images`` (default range(N))."""
    images = list(range(N)) if images is None else list(images)
    L = len(shapes)
    S = sum(h * w for h, w in shapes)
    dt = DTYPES[dtype]

    def stack(fn, shape):
        if not images:
            return torch.empty((0,) + shape, dtype=dt)
        return torch.stack([fn(n) for n in images]).to(dt)

    value = stack(lambda n: _uniform((S, M, D), seed_of(TENSOR_VALUE, n), -1.0, 1.0), (S, M, D))
    loc = stack(lambda n: _uniform((Lq, M, L, P, 2), seed_of(TENSOR_LOC, n), *loc_range),
                (Lq, M, L, P, 2))
    attn = stack(lambda n: _uniform((Lq, M, L, P), seed_of(TENSOR_ATTN, n), 0.0, 2.0 / (L * P)),
                 (Lq, M, L, P))
    gout = stack(lambda n: _uniform((Lq, M, D), seed_of(TENSOR_GOUT, n), -1.0, 1.0),
                 (Lq, M, D)) if with_gout else None
    return value, loc, attn, gout


# ---------------------------------------------------------------------------------------
# Module-path inputs (NEXT-2, R21): the fused offset/mask
# linear layer's parameters, drawn like a trained layer's scale so that its
# outputs land in the operator's working ranges for x ~ U(-1, 1):
#   weight [J, C], J = 3*G*K: offset rows ~ U(-1, 1) * 2*sqrt(3/C) (offsets of std
#   ~1.15 px), mask rows ~ U(-1, 1) * sqrt(3/C) (std ~0.58);  bias ~ U(-0.5, 0.5).
TENSOR_WEIGHT, TENSOR_BIAS = 20, 21


def make_linear(C, G, K, dtype="f32", seed=0):
    """CPU tensors (weight [3GK, C], bias [3GK]) in ``dtype``."""
    J = 3 * G * K
    g = torch.Generator().manual_seed(seed_of(TENSOR_WEIGHT, seed))
    w = (torch.rand((J, C), generator=g, dtype=torch.float32) * 2.0 - 1.0) * (3.0 / C) ** 0.5
    scale = torch.ones(G, 3 * K)
    scale[:, : 2 * K] = 2.0
    w = w * scale.reshape(J, 1)
    g = torch.Generator().manual_seed(seed_of(TENSOR_BIAS, seed))
    b = torch.rand((J,), generator=g, dtype=torch.float32) - 0.5
    return w.to(DTYPES[dtype]), b.to(DTYPES[dtype])


# Full-module projections (NEXT-2, R22): the 1x1 input / output projections of
# P:198 drawn like an initialised layer, weight [C_out, C_in] ~ U(-1, 1) * sqrt(3 / C_in)
# (unit-variance outputs for unit-variance inputs), bias ~ U(-0.1, 0.1).
TENSOR_PROJ_W, TENSOR_PROJ_B = 22, 23


def make_projection(C_out, C_in, dtype="f32", seed=0):
    """CPU tensors (weight [C_out, C_in], bias [C_out]) in ``dtype``."""
    g = torch.Generator().manual_seed(seed_of(TENSOR_PROJ_W, seed))
    w = (torch.rand((C_out, C_in), generator=g, dtype=torch.float32) * 2.0 - 1.0) * (3.0 / C_in) ** 0.5
    g = torch.Generator().manual_seed(seed_of(TENSOR_PROJ_B, seed))
    b = (torch.rand((C_out,), generator=g, dtype=torch.float32) * 2.0 - 1.0) * 0.1
    return w.to(DTYPES[dtype]), b.to(DTYPES[dtype])


def make_module_params(C, G, K=9, dtype="f32", seed=0):
    """The full module's parameters {w_in, b_in, w_om, b_om, w_out, b_out} (CPU)."""
    w_in, b_in = make_projection(C, C, dtype, 2 * seed)
    w_out, b_out = make_projection(C, C, dtype, 2 * seed + 1)
    w_om, b_om = make_linear(C, G, K, dtype, seed)
    return {"w_in": w_in, "b_in": b_in, "w_om": w_om, "b_om": b_om, "w_out": w_out, "b_out": b_out}
