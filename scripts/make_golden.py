"""Freeze the oracle's outputs on BASELINE.json config c1 (tiny fp32 fwd+bwd) into
tests/golden/c1_tiny.json ("freeze on first run"; a regression guard
against later oracle edits, not a truth source).  Calls only oracle/ and synth/."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    g = oracle.Geometry(N=1, H=8, W=8, G=2, D=16)
    Ho, Wo = g.out_hw()
    x, om, gy = synth.make_case(1, 8, 8, 2, 16, Ho, Wo, 9, g.S, "f32")
    y = oracle.forward(g, x, om)
    gx, gom = oracle.backward(g, x, om, gy)
    out = {
        "citation": "BASELINE.json configs[0] (c1): N=1, H=W=8, G=2, D=16, 3x3, stride 1, "
                    "pad 1, fp32 inputs from synth (seeds 20240111 + 1000*tensor + image). "
                    "Values written by scripts/make_golden.py from oracle/ only.",
        "inputs_sha256": {k: hashlib.sha256(t.numpy().tobytes()).hexdigest()
                          for k, t in (("x", x), ("om", om), ("gy", gy))},
        "y": [float.hex(float(v)) for v in y.ravel()],
        "grad_x": [float.hex(float(v)) for v in gx.ravel()],
        "grad_om": [float.hex(float(v)) for v in gom.ravel()],
    }
    path = os.path.join(ROOT, "tests", "golden", "c1_tiny.json")
    if os.path.exists(path) and "--force" not in sys.argv:
        print(f"{path} exists; refusing to overwrite without --force")
        return 2
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path)
    return 0


if __name__ == "__main__":
    sys.exit(main())
