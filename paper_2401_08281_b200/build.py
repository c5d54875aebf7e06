"""Build libflatknn.so in-tree with nvcc for sm_100a.

    python -m paper_2401_08281_b200.build

The shared library is the C-ABI boundary declared in ``include/flatknn.h``;
it statically links the CUDA runtime so the only runtime dependency is the
driver (libcuda), which ctypes loads alongside torch's own runtime.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_NAME = "libflatknn.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)
# development variant (clock64 timeline trace + bottleneck flags, -DFK_DEV=1):
# loaded instead of the product library only when FK_DEV_LIB=1 (scripts/)
DEV_LIB_PATH = os.path.join(PKG_DIR, "libflatknn_dev.so")

SOURCES = ["flatknn.cu"]
DEPS = SOURCES + ["flatknn_kernels.cuh", "sm100.cuh"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build(path: str = LIB_PATH) -> bool:
    if not os.path.exists(path):
        return True
    t = os.path.getmtime(path)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(REPO, "include", "flatknn.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = True, dev: bool = False) -> str:
    out = DEV_LIB_PATH if dev else LIB_PATH
    if not force and not needs_build(out):
        return out
    cmd = [
        nvcc_path(),
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
        "-Xptxas", "-v",
        "-I", os.path.join(REPO, "include"),
        "-o", out + ".tmp",
    ] + (["-DFK_DEV=1"] if dev else []) + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        print("[build]", " ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    log_path = os.path.join(PKG_DIR, "build_dev.log" if dev else "build.log")
    with open(log_path, "w") as f:
        f.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed (see {log_path}):\n{res.stderr[-4000:]}")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, dev="--dev" in sys.argv))
