"""Mutation check of the oracle's pins: copy oracle/, tests/, synth/ and
the package to a scratch directory, apply one plausible mistake at a time to the fp64 C
oracle -- inflated magnitude scales, a dropped term, a wrong sign, a swapped axis -- and
run the CPU pin tests against it.  Every mutation must fail at least one test.

  python scripts/oracle_mutations.py [--out profiles/r02_oracle_mutations.txt]
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, original text, mutated text) in oracle/dcnv4_oracle.c
MUTATIONS = [
    ("grad_dy magnitude scale x50", "garow[2 * k + 1] = fabs(s * m[k]) * agy;",
     "garow[2 * k + 1] = 50.0 * fabs(s * m[k]) * agy;"),
    ("grad_dx magnitude scale x50", "garow[2 * k] = fabs(s * m[k]) * agx;",
     "garow[2 * k] = 50.0 * fabs(s * m[k]) * agx;"),
    ("softmax grad_mask magnitude scale x100", "garow[2 * K + k] = m[k] * (gma[k] + adot);",
     "garow[2 * K + k] = 100.0 * m[k] * (gma[k] + adot);"),
    ("grad_mask magnitude scale x50", "gma[k] = agm;", "gma[k] = 50.0 * agm;"),
    ("grad_input magnitude scale x50", "gx_abs[q] += fabs(m[k]) * cw[corner] * fabs(g_y[c]);",
     "gx_abs[q] += 50.0 * fabs(m[k]) * cw[corner] * fabs(g_y[c]);"),
    ("grad_dy sign", "grow[2 * k + 1] = s * m[k] * sgy;", "grow[2 * k + 1] = -s * m[k] * sgy;"),
    ("grad_dx without offset_scale", "grow[2 * k] = s * m[k] * sgx;", "grow[2 * k] = m[k] * sgx;"),
    ("grad_input drops m", "gx[q] += m[k] * cw[corner] * g_y[c];", "gx[q] += cw[corner] * g_y[c];"),
    ("softmax Jacobian sign", "grow[2 * K + k] = m[k] * (gm[k] - dot);",
     "grow[2 * K + k] = m[k] * (gm[k] + dot);"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--only", default="", help="run only the mutation with this name")
    args = ap.parse_args()
    muts = [m for m in MUTATIONS if not args.only or m[0] == args.only]
    if not muts:
        raise SystemExit(f"no mutation named {args.only!r}")
    lines = []
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "tests", "synth", "paper_2401_06197_b200"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("build", "*.so", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        src = os.path.join(tmp, "oracle", "dcnv4_oracle.c")
        base = open(src).read()
        ok = True
        for name, a, b in muts:
            if a not in base:
                lines.append(f"{name}: PATTERN NOT FOUND")
                ok = False
                continue
            with open(src, "w") as f:
                f.write(base.replace(a, b))
            for f in os.listdir(os.path.join(tmp, "oracle")):
                if f.endswith(".so"):
                    os.remove(os.path.join(tmp, "oracle", f))
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py",
                                "tests/test_golden.py", "tests/test_oracle_module_full.py", "-q", "-m", "not gpu",
                                "-p", "no:cacheprovider"], cwd=tmp, capture_output=True, text=True)
            last = (r.stdout.strip().splitlines() or ["?"])[-1]
            caught = r.returncode != 0
            ok &= caught
            lines.append(f"{'caught' if caught else 'MISSED'}  {name}: {last}")
        with open(src, "w") as f:
            f.write(base)
    report = "\n".join(lines) + ("\nall mutations caught\n" if ok else "\nSOME MUTATIONS MISSED\n")
    print(report, end="")
    if args.out:
        with open(args.out, "w") as f:
            f.write("# scripts/oracle_mutations.py: one mutation of oracle/dcnv4_oracle.c at a time vs the CPU pins\n")
            f.write(report)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
