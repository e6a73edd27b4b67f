"""Regression freeze of the oracle on config c1 (written by scripts/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c1_tiny.json")


def test_c1_tiny_frozen_outputs():
    with open(GOLDEN) as f:
        fx = json.load(f)
    g = oracle.Geometry(N=1, H=8, W=8, G=2, D=16)
    Ho, Wo = g.out_hw()
    x, om, gy = synth.make_case(1, 8, 8, 2, 16, Ho, Wo, 9, g.S, "f32")
    for k, t in (("x", x), ("om", om), ("gy", gy)):
        assert hashlib.sha256(t.numpy().tobytes()).hexdigest() == fx["inputs_sha256"][k], k
    y = oracle.forward(g, x, om)
    gx, gom = oracle.backward(g, x, om, gy)
    for name, arr in (("y", y), ("grad_x", gx), ("grad_om", gom)):
        ref = np.array([float.fromhex(v) for v in fx[name]])
        np.testing.assert_allclose(arr.ravel(), ref, rtol=0, atol=1e-14)
