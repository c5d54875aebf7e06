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

# one translation unit per fused-kernel operand MODE (the template
# instantiations dominate compile time) + the host/ABI unit; compiled in
# parallel, linked into one shared library
SOURCES = ["flatknn.cu", "xchg.cu"] + [f"fused_m{m}.cu" for m in range(6)]
DEPS = SOURCES + ["flatknn_kernels.cuh", "fused_kernel.cuh", "fused_launch.cuh", "fk_host.cuh", "sm100.cuh", "storage_kernels.cuh", "filter16_kernels.cuh"]


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


def variant_path(name: str) -> str:
    return os.path.join(PKG_DIR, f"libflatknn_{name}.so")


def build(force: bool = False, verbose: bool = True, dev: bool = False, variant: str | None = None,
          defines: tuple = ()) -> str:
    """variant/defines: an experiment library libflatknn_<variant>.so built with
    extra -D flags (loaded only with FK_LIB_VARIANT=<variant>, scripts only)."""
    out = variant_path(variant) if variant else (DEV_LIB_PATH if dev else LIB_PATH)
    if not force and not needs_build(out):
        return out
    nvcc = nvcc_path()
    common = [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17",
        "-Xcompiler", "-fPIC,-O3",
        "-Xptxas", "-v",
        "-I", os.path.join(REPO, "include"),
    ] + (["-DFK_DEV=1"] if dev else []) + [f"-D{d}" for d in defines]
    objdir = os.path.join(PKG_DIR, f"_obj_{variant}" if variant else ("_obj_dev" if dev else "_obj"))
    os.makedirs(objdir, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc, "-c"] + common + ["-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print("[build]", " ".join(cmd), file=sys.stderr)
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    logs, failed = [], []
    for src, obj, pr in procs:
        text = pr.communicate()[0]
        logs.append(f"==== {src}\n{text}")
        if pr.returncode != 0:
            failed.append(src)
    log_path = os.path.join(PKG_DIR, f"build_{variant}.log" if variant else ("build_dev.log" if dev else "build.log"))
    with open(log_path, "w") as f:
        f.write("\n".join(logs))
    if failed:
        raise RuntimeError(f"nvcc failed for {failed} (see {log_path}):\n" + "\n".join(logs)[-4000:])
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
            "-o", out + ".tmp"] + [obj for _, obj, _ in procs]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, dev="--dev" in sys.argv))
