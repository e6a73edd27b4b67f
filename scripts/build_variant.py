"""Build an A/B variant of libdcnv4.so with extra -D defines (compile-time experiment knobs,
e.g. DCNV4_PULL_PC in csrc/dcnv4_kernels.cuh).  Only the translation units named with
--tu are recompiled with the defines (and DCNV4_VARIANT_MIN: only the D = 16 fp32 /
half instantiations, for compile time); the rest are linked from the in-tree build.

  python scripts/build_variant.py --name pc1 --tu dcnv4_f32.cu -D DCNV4_PULL_PC=1
  DCNV4_LIB=$PWD/build_variants/pc1/libdcnv4.so python scripts/tune.py ...
"""
import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2401_06197_b200 import _build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", required=True)
    ap.add_argument("--tu", action="append", default=[])
    ap.add_argument("-D", dest="defs", action="append", default=[])
    args = ap.parse_args()
    # the other translation units are linked from the in-tree build as they are (built
    # once if missing); compare variants against a variant built with no -D ("base")
    if not all(os.path.exists(os.path.join(_build.BUILD, s.replace(".cu", ".o"))) for s in _build.SOURCES):
        _build.build(verbose=False)
    out = os.path.join(ROOT, "build_variants", args.name)
    os.makedirs(out, exist_ok=True)
    defs = ["-DDCNV4_VARIANT_MIN"] + [f"-D{d}" for d in args.defs]

    def comp(tu):
        obj = os.path.join(out, tu.replace(".cu", ".o"))
        cmd = [_build.NVCC, *_build.ARCH, *_build.FLAGS, *defs, "-c", os.path.join(_build.CSRC, tu), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(obj + ".ptxas.log", "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode:
            raise SystemExit(f"nvcc failed for {tu}:\n{r.stderr[-3000:]}")
        return obj

    # the host planner (shared-memory carve-up, launch shapes) always follows the kernels
    if "dcnv4_api.cu" not in args.tu:
        args.tu.append("dcnv4_api.cu")
    with cf.ThreadPoolExecutor(max(1, len(args.tu))) as ex:
        new = dict(zip(args.tu, ex.map(comp, args.tu)))
    objs = [new.get(s, os.path.join(_build.BUILD, s.replace(".cu", ".o"))) for s in _build.SOURCES]
    lib = os.path.join(out, "libdcnv4.so")
    subprocess.check_call([_build.NVCC, *_build.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs])
    print(lib)


if __name__ == "__main__":
    main()
