"""Build libdcnv4.so in-tree with nvcc for sm_100a (no torch JIT, no cache outside the repo)."""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libdcnv4.so")
SOURCES = ["dcnv4_api.cu", "dcnv4_f32.cu", "dcnv4_f16.cu", "dcnv4_bf16.cu", "msda.cu", "om_linear.cu", "module_fwd.cu", "gemm.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v", "-Xcompiler", "-Wall"]


def _source_hash() -> str:
    """sha256 over every CUDA source/header, the ABI headers and the compiler command: the
    library is rebuilt whenever any of them differs from what the in-tree .so was built
    from (not by mtime, so a stale prebuilt binary never stands in for HEAD)."""
    h = hashlib.sha256()
    files = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC))
    for name in ("dcnv4.h", "msda.h", "dcnv4_module.h"):
        files.append(os.path.join(os.path.dirname(HERE), "include", name))
    for f in files:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join([NVCC, *ARCH, *FLAGS, *SOURCES]).encode())
    return h.hexdigest()


STAMP = os.path.join(BUILD, "libdcnv4.sha256")


def _object_hash(src: str) -> str:
    """sha256 of one translation unit: its source, every header it may include, the flags."""
    h = hashlib.sha256()
    with open(os.path.join(CSRC, src), "rb") as fh:
        h.update(fh.read())
    hdrs = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))
    hdrs += [os.path.join(os.path.dirname(HERE), "include", n) for n in ("dcnv4.h", "msda.h", "dcnv4_module.h")]
    for f in hdrs:
        with open(f, "rb") as fh:
            h.update(fh.read())
    h.update(" ".join([NVCC, *ARCH, *FLAGS]).encode())
    return h.hexdigest()


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    log = os.path.join(BUILD, src.replace(".cu", ".ptxas.log"))
    stamp = obj + ".sha256"
    digest = _object_hash(src)
    if os.path.exists(obj) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == digest:
                return obj  # unchanged translation unit
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    with open(stamp, "w") as f:
        f.write(digest + "\n")
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    digest = _source_hash()
    if not force and os.path.exists(LIB) and os.path.exists(STAMP):
        with open(STAMP) as f:
            if f.read().strip() == digest:
                return LIB
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(digest + "\n")
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
