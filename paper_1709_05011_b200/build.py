"""Build the CUDA C-ABI library in-tree (nvcc, sm_100a only).

`python -m paper_1709_05011_b200.build` (or `__graft_entry__.build()`)
produces `paper_1709_05011_b200/_lib/liblars_b200.so`.  The library links
cudart statically and exports only the `extern "C"` symbols of
`include/lars_b200.h`, so it loads on a machine without a GPU (the CPU tests
check the exports) and on the B200 box it shares the primary context with
PyTorch.
"""

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = os.path.join(PKG, "csrc", "lars_kernels.cu")
INCLUDE = os.path.join(ROOT, "include")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "liblars_b200.so")
TRACE_LIB = os.path.join(LIB_DIR, "liblars_b200_trace.so")  # -DLARS_TRACE, profiling only

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-shared", "--cudart", "static",
]


def nvcc():
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found")
    return path


def sources():
    return [SRC, os.path.join(INCLUDE, "lars_b200.h")]


def up_to_date(lib=LIB):
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force=False, verbose=False, trace=False):
    lib = TRACE_LIB if trace else LIB
    if not force and up_to_date(lib):
        return lib
    os.makedirs(LIB_DIR, exist_ok=True)
    tmp = lib + ".tmp"
    extra = ["-DLARS_TRACE"] if trace else []
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", INCLUDE, SRC, "-o", tmp]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
    os.replace(tmp, lib)
    if verbose:
        sys.stdout.write(proc.stderr)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
