"""fp64 CPU oracle for the DCNv4 spatial aggregation -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg
and ``--impl reference``) may import this package.  The product path
(``paper_2401_06197_b200``) never imports it, and this package imports nothing from
the product path: the two share no code.

The arithmetic lives in ``dcnv4_oracle.c`` (plain C, fp64, OpenMP over (n, g)); this
module only builds it with gcc, marshals numpy arrays, and converts stored values
exactly to fp64.  Every function cites the passage it follows:

* forward  -- PAPER.md Eq. (1)-(2), softmax removed;
* backward -- Eq. (1) differentiated, right derivative at kinks;
* softmax  -- the DCNv3 normalisation over K, behind ``softmax=True``.

Parity status: every output is pinned (tests/test_oracle_pins.py); see DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dcnv4_oracle.c")
_LIB = os.path.join(_HERE, "libdcnv4_oracle.so")
_MSRC = os.path.join(_HERE, "msda_oracle.c")
_MLIB = os.path.join(_HERE, "libmsda_oracle.so")
_lib = None
_mlib = None


def _gcc(src: str, lib: str, force: bool) -> str:
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        tmp = lib + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
             "-shared", "-fPIC", "-o", tmp, src, "-lm"])
        os.replace(tmp, lib)
    return lib


def build(force: bool = False) -> str:
    """Compile the oracles with gcc (fp64, no fast-math, no FMA contraction)."""
    _gcc(_MSRC, _MLIB, force)
    return _gcc(_SRC, _LIB, force)


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        lib.oracle_output_size.argtypes = [P, P, P]
        lib.oracle_forward.argtypes = [P, ctypes.c_double, P, P, P, P]
        lib.oracle_backward.argtypes = [P, ctypes.c_double, P, P, P, P, P, P, P]
        lib.oracle_forward.restype = ctypes.c_int
        lib.oracle_backward.restype = ctypes.c_int
        lib.oracle_output_size.restype = ctypes.c_int
        lib.oracle_geom_len.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass(frozen=True)
class Geometry:
    """Problem geometry (Eq. (1): x in R^{HxWxC}, G groups, K = kh*kw points).

    ``om_stride`` is S, the channel count of one offset_mask row (0 -> 3*G*K)."""
    N: int
    H: int
    W: int
    G: int
    D: int
    kh: int = 3
    kw: int = 3
    sh: int = 1
    sw: int = 1
    ph: int = 1
    pw: int = 1
    dh: int = 1
    dw: int = 1
    offset_scale: float = 1.0
    om_stride: int = 0
    softmax: bool = False

    @property
    def K(self) -> int:
        return self.kh * self.kw

    @property
    def C(self) -> int:
        return self.G * self.D

    @property
    def S(self) -> int:
        return self.om_stride if self.om_stride else 3 * self.G * self.K

    def out_hw(self):
        # conv2d output arithmetic (reading R4, "as in regular convolutions")
        Ho = (self.H + 2 * self.ph - self.dh * (self.kh - 1) - 1) // self.sh + 1
        Wo = (self.W + 2 * self.pw - self.dw * (self.kw - 1) - 1) // self.sw + 1
        return Ho, Wo

    def vec(self) -> np.ndarray:
        return np.array([self.N, self.H, self.W, self.G, self.D, self.kh, self.kw, self.sh,
                         self.sw, self.ph, self.pw, self.dh, self.dw, self.S,
                         int(self.softmax)], dtype=np.int64)


def _f64(a) -> np.ndarray:
    """Exact conversion of stored fp32/fp16/bf16 values to a contiguous fp64 array."""
    if hasattr(a, "detach"):  # torch tensor: .double() is exact for fp32/fp16/bf16
        a = a.detach().to("cpu").double().numpy()
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def forward(geom: Geometry, x, om, with_abs: bool = False):
    """y = DCNv4(x, offset_mask) in fp64 (Eq. (1)-(2)).  Returns y or (y, y_abs)."""
    lib = _load()
    Ho, Wo = geom.out_hw()
    x = _f64(x).reshape(geom.N, geom.H, geom.W, geom.C)
    om = _f64(om).reshape(geom.N, Ho, Wo, geom.S)
    y = np.empty((geom.N, Ho, Wo, geom.C), np.float64)
    ya = np.empty_like(y) if with_abs else None
    gv = geom.vec()
    rc = lib.oracle_forward(_ptr(gv), geom.offset_scale, _ptr(x), _ptr(om), _ptr(y),
                            _ptr(ya) if with_abs else None)
    if rc:
        raise ValueError(f"oracle_forward failed with code {rc}")
    return (y, ya) if with_abs else y


def backward(geom: Geometry, x, om, gy, with_abs: bool = False):
    """(grad_x, grad_om) of Eq. (1) in fp64; with_abs adds their magnitude scales."""
    lib = _load()
    Ho, Wo = geom.out_hw()
    x = _f64(x).reshape(geom.N, geom.H, geom.W, geom.C)
    om = _f64(om).reshape(geom.N, Ho, Wo, geom.S)
    gy = _f64(gy).reshape(geom.N, Ho, Wo, geom.C)
    gx = np.empty_like(x)
    gom = np.empty_like(om)
    gxa = np.empty_like(x) if with_abs else None
    goma = np.empty_like(om) if with_abs else None
    gv = geom.vec()
    rc = lib.oracle_backward(_ptr(gv), geom.offset_scale, _ptr(x), _ptr(om), _ptr(gy),
                             _ptr(gx), _ptr(gom), _ptr(gxa) if with_abs else None,
                             _ptr(goma) if with_abs else None)
    if rc:
        raise ValueError(f"oracle_backward failed with code {rc}")
    return (gx, gom, gxa, goma) if with_abs else (gx, gom)


def abs_scaled_error(gpu, ref, scale) -> float:
    """max_i |gpu_i - ref_i| / (A_i + 1e-30 * max A)  (SURVEY 8(c).4 metric)."""
    gpu = _f64(gpu)
    ref = _f64(ref)
    scale = _f64(scale)
    den = scale + max(1e-30 * float(scale.max(initial=0.0)), 1e-300)
    if gpu.size == 0:
        return 0.0
    return float((np.abs(gpu - ref) / den).max())


# ---------------------------------------------------------------------------------------
# Multi-scale deformable attention (R20).  The paper names
# the operator and says the DCNv4 kernel techniques apply to it; the
# sampling core is written out in msda_oracle.c.


@dataclass(frozen=True)
class MSDAGeometry:
    """value [N][S][M][D] over levels `shapes` = ((H_0, W_0), ...), S = sum H_l*W_l;
    loc [N][Lq][M][L][P][2] (x, y) in [0, 1]; attn [N][Lq][M][L][P]."""
    N: int
    Lq: int
    M: int
    D: int
    P: int
    shapes: tuple

    @property
    def L(self) -> int:
        return len(self.shapes)

    @property
    def S(self) -> int:
        return sum(h * w for h, w in self.shapes)

    def vec(self) -> np.ndarray:
        v = [self.N, self.Lq, self.M, self.D, self.L, self.P]
        for h, w in self.shapes:
            v += [h, w]
        return np.array(v, dtype=np.int64)


def _mload():
    global _mlib
    if _mlib is None:
        build()
        lib = ctypes.CDLL(_MLIB)
        P = ctypes.c_void_p
        lib.msda_oracle_forward.argtypes = [P] * 6
        lib.msda_oracle_backward.argtypes = [P] * 11
        lib.msda_oracle_forward.restype = ctypes.c_int
        lib.msda_oracle_backward.restype = ctypes.c_int
        _mlib = lib
    return _mlib


def msda_forward(geom: MSDAGeometry, value, loc, attn, with_abs: bool = False):
    """out [N][Lq][M][D] in fp64 (msda_oracle.c header).  Returns out or (out, out_abs)."""
    lib = _mload()
    g = geom
    value = _f64(value).reshape(g.N, g.S, g.M, g.D)
    loc = _f64(loc).reshape(g.N, g.Lq, g.M, g.L, g.P, 2)
    attn = _f64(attn).reshape(g.N, g.Lq, g.M, g.L, g.P)
    out = np.empty((g.N, g.Lq, g.M, g.D), np.float64)
    oa = np.empty_like(out) if with_abs else None
    gv = g.vec()
    lib.msda_oracle_forward(_ptr(gv), _ptr(value), _ptr(loc), _ptr(attn), _ptr(out),
                            _ptr(oa) if with_abs else None)
    return (out, oa) if with_abs else out


def msda_backward(geom: MSDAGeometry, value, loc, attn, gout, with_abs: bool = False):
    """(grad_value, grad_loc, grad_attn) in fp64; with_abs adds their magnitude scales."""
    lib = _mload()
    g = geom
    value = _f64(value).reshape(g.N, g.S, g.M, g.D)
    loc = _f64(loc).reshape(g.N, g.Lq, g.M, g.L, g.P, 2)
    attn = _f64(attn).reshape(g.N, g.Lq, g.M, g.L, g.P)
    gout = _f64(gout).reshape(g.N, g.Lq, g.M, g.D)
    gval = np.empty_like(value)
    gloc = np.empty_like(loc)
    gattn = np.empty_like(attn)
    ab = [np.empty_like(a) for a in (gval, gloc, gattn)] if with_abs else [None] * 3
    gv = g.vec()
    lib.msda_oracle_backward(_ptr(gv), _ptr(value), _ptr(loc), _ptr(attn), _ptr(gout),
                             _ptr(gval), _ptr(gloc), _ptr(gattn),
                             *[(_ptr(a) if a is not None else None) for a in ab])
    return (gval, gloc, gattn, *ab) if with_abs else (gval, gloc, gattn)


# ---------------------------------------------------------------------------------------
# DCNv4 module path (R21).  P:334: "the linear layers for
# computing offset and dynamic weights can actually be combined into one linear layer",
# and the depthwise conv in front of it "can also be removed" (latency-first variant);
# the "lightweight" module has no input/output projections, so the value
# the operator samples is the module input itself.  Reading R21: the linear's output is
# stored in the storage dtype T before the operator reads it (what an unfused module
# holds between its two layers), so the oracle rounds it once, fp64 -> T, RN-even.

_ROUND = {"f32": (24, -125, 3.4028234663852886e38), "f16": (11, -13, 65504.0),
          "bf16": (8, -125, 3.3895313892515355e38)}


def round_to(v, dtype: str) -> np.ndarray:
    """Round fp64 values to the nearest `dtype` value (ties to even), subnormals and
    overflow to +-inf included.  v = m * 2^e with m in [0.5, 1): the quantum is
    2^(max(e, emin) - p) for p significant bits; np.rint rounds half to even."""
    p, emin, vmax = _ROUND[dtype]
    v = np.asarray(v, dtype=np.float64)
    _, e = np.frexp(v)
    q = np.ldexp(1.0, np.maximum(e, emin) - p)
    r = np.rint(v / q) * q
    # |v| at or beyond the rounding midpoint above the largest finite value -> inf
    big = np.abs(v) >= vmax + np.ldexp(1.0, np.frexp(vmax)[1] - p - 1)
    return np.where(big, np.copysign(np.inf, v), r)


def offset_mask_linear(feat, weight, bias, S: int, dtype: str = "f32", with_abs: bool = False):
    """om[r, j] = round_T(sum_c feat[r, c] * weight[j, c] + bias[j]) for j < J = weight
    rows (= 3GK), om[r, j] = 0 for J <= j < S (reading R21).

    feat [R, C_in], weight [J, C_in], bias [J] (or None).  The contraction is one fp64
    matrix product (a library primitive standing for the linear layer's definition).
    Returns om (fp64 holding T values) or, with_abs, (om, om_exact, om_abs) where
    om_exact is the unrounded fp64 result and om_abs = |feat| @ |weight|^T + |bias|."""
    f = _f64(feat)
    w = _f64(weight)
    R, J = f.shape[0], w.shape[0]
    b = np.zeros(J) if bias is None else _f64(bias).reshape(J)
    exact = np.zeros((R, S))
    exact[:, :J] = f @ w.T + b
    om = round_to(exact, dtype)
    if not with_abs:
        return om
    ab = np.zeros((R, S))
    ab[:, :J] = np.abs(f) @ np.abs(w).T + np.abs(b)
    return om, exact, ab


def module_forward(geom: Geometry, x, weight, bias, dtype: str = "f32", with_abs: bool = False):
    """Lightweight DCNv4 module forward: om = offset_mask_linear(x)
    at every output pixel (stride 1, 'same' output, so the linear reads x[n, ho, wo]),
    then y = DCNv4(x, om) (Eq. (1)-(2)).  Returns y, or (y, y_abs, om)."""
    Ho, Wo = geom.out_hw()
    if (Ho, Wo) != (geom.H, geom.W):
        raise ValueError("module_forward needs Ho == H and Wo == W (the linear reads x per pixel)")
    xf = _f64(x).reshape(geom.N * geom.H * geom.W, geom.C)
    om = offset_mask_linear(xf, weight, bias, geom.S, dtype)
    om = om.reshape(geom.N, Ho, Wo, geom.S)
    if not with_abs:
        return forward(geom, xf, om)
    y, ya = forward(geom, xf, om, with_abs=True)
    return y, ya, om


# ---------------------------------------------------------------------------------------
# The full DCNv4 module (R21, R22).  P:198: "A 1x1
# point-wise convolution on x and y can be applied before and after" the spatial
# aggregation; the offsets and aggregation weights come from one linear layer;
# this full module (with the projections) is the one used in the rest of the
# models.  Reading R22: the projected value v = x W_in^T + b_in is what the operator
# samples, while the offset/mask linear reads the module input x (prior-art DCNv3/v4
# module wiring; the paper does not draw the module).  Every layer's output is stored in
# the storage dtype T between layers (R21 extended: what an unfused module holds in
# memory), so each is rounded once, fp64 -> T.  dtype "f64" disables the rounding.

def _rt(v, dtype):
    return np.asarray(v, dtype=np.float64) if dtype == "f64" else round_to(v, dtype)


def linear(x, weight, bias=None, dtype: str = "f64"):
    """y = round_T(x @ weight^T + bias): nn.Linear / a 1x1 convolution in fp64.
    x [R, K], weight [N, K], bias [N] or None."""
    x, w = _f64(x), _f64(weight)
    y = x @ w.T
    if bias is not None:
        y = y + _f64(bias).reshape(1, -1)
    return _rt(y, dtype)


def linear_abs(x_abs, weight, bias=None):
    """Magnitude scale of linear(): |x| @ |W|^T + |b| (SURVEY 8(c).4 metric, chained)."""
    y = _f64(x_abs) @ np.abs(_f64(weight)).T
    if bias is not None:
        y = y + np.abs(_f64(bias)).reshape(1, -1)
    return y


def module_full_forward(geom: Geometry, x, params: dict, dtype: str = "f64", with_abs: bool = False):
    """Full DCNv4 module forward: v = linear(x; W_in, b_in), om = linear(x; W_om, b_om)
    (padded to S channels with zeros), a = DCNv4(v, om) (Eq. (1)-(2)),
    y = linear(a; W_out, b_out); each output rounded to T (R22).  params: w_in, b_in,
    w_om, b_om, w_out, b_out (biases may be None).  Stride-1 'same' geometry.
    Returns a dict with v, om, a, y (fp64 arrays in NHWC) and, with_abs, y_abs / a_abs."""
    Ho, Wo = geom.out_hw()
    if (Ho, Wo) != (geom.H, geom.W):
        raise ValueError("the full module needs Ho == H and Wo == W")
    R = geom.N * geom.H * geom.W
    xf = _f64(x).reshape(R, geom.C)
    v = linear(xf, params["w_in"], params.get("b_in"), dtype)
    J = _f64(params["w_om"]).shape[0]
    om = np.zeros((R, geom.S))
    om[:, :J] = linear(xf, params["w_om"], params.get("b_om"), dtype)
    om = om.reshape(geom.N, Ho, Wo, geom.S)
    out = {"v": v.reshape(geom.N, geom.H, geom.W, geom.C), "om": om}
    if with_abs:
        a, a_abs0 = forward(geom, v, om, with_abs=True)
        v_abs = linear_abs(np.abs(xf), params["w_in"], params.get("b_in"))
        # DCNv4 magnitude pass over the value magnitudes: sum |m| w v_abs
        _, a_abs = forward(geom, v_abs, om, with_abs=True)
        a = _rt(a, dtype)
        out["a_abs"] = a_abs
        out["y_abs"] = linear_abs(a_abs.reshape(R, geom.C), params["w_out"], params.get("b_out")).reshape(
            geom.N, Ho, Wo, -1)
    else:
        a = _rt(forward(geom, v, om), dtype)
    out["a"] = a
    out["y"] = linear(a.reshape(R, geom.C), params["w_out"], params.get("b_out"), dtype).reshape(
        geom.N, Ho, Wo, -1)
    return out


def module_full_backward(geom: Geometry, x, params: dict, gy, dtype: str = "f64"):
    """Backward of module_full_forward given gy = dL/dy, each stored result rounded to T
    (R22): ga = gy @ W_out, (gv, gom) = DCNv4 backward, and for each
    linear y = x W^T + b: dx = dy @ W, dW = dy^T @ x, db = sum_rows dy.  The module input
    feeds both the input projection and the offset/mask linear, so
    gx = gv @ W_in + gom[:, :J] @ W_om.  Returns a dict of fp64 arrays."""
    fw = module_full_forward(geom, x, params, dtype)
    R = geom.N * geom.H * geom.W
    xf = _f64(x).reshape(R, geom.C)
    gyf = _f64(gy).reshape(R, -1)
    a = fw["a"].reshape(R, geom.C)
    w_out, w_in, w_om = _f64(params["w_out"]), _f64(params["w_in"]), _f64(params["w_om"])
    J = w_om.shape[0]
    g = {}
    g["w_out"] = _rt(gyf.T @ a, dtype)
    g["b_out"] = _rt(gyf.sum(axis=0), dtype)
    ga = _rt(gyf @ w_out, dtype)
    gv, gom = backward(geom, fw["v"], fw["om"], ga.reshape(geom.N, geom.H, geom.W, geom.C))
    gv = _rt(gv.reshape(R, geom.C), dtype)
    gom = _rt(gom.reshape(R, geom.S), dtype)
    g["w_in"] = _rt(gv.T @ xf, dtype)
    g["b_in"] = _rt(gv.sum(axis=0), dtype)
    g["w_om"] = _rt(gom[:, :J].T @ xf, dtype)
    g["b_om"] = _rt(gom[:, :J].sum(axis=0), dtype)
    g["x"] = _rt(gv @ w_in + gom[:, :J] @ w_om, dtype).reshape(geom.N, geom.H, geom.W, geom.C)
    g["a"] = ga.reshape(geom.N, geom.H, geom.W, geom.C)
    g["v"] = gv.reshape(geom.N, geom.H, geom.W, geom.C)
    g["om"] = gom.reshape(geom.N, geom.H, geom.W, geom.S)
    return g
