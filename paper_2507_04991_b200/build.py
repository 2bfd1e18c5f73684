"""Build the in-tree CUDA library libperrk_b200.so (sm_100a, -lineinfo).

The library holds the device kernels (csrc/dg_kernels.cu) and the C++ host
layer + C-ABI (csrc/host.cpp, include/perrk_b200.h).  It is built in place so
the .so travels with the repository snapshot to the GPU host.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libperrk_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["dg_kernels.cu", "host.cpp"]
DEPS = SOURCES + ["dg_device.cuh", "dg_launch.hpp", "dg_stage.cuh", "dg_stage3w.cuh", "dg_stage2w.cuh", "dg_visc.cuh", "dg_advection.cuh", "dg_krylov.cuh"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    files = [os.path.join(CSRC, f) for f in DEPS] + [
        os.path.join(ROOT, "include", "perrk_b200.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(f) > t for f in files)


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"),
           *os.environ.get("PERRK_NVCC_FLAGS", "").split(),
           *[os.path.join(CSRC, f) for f in SOURCES],
           "-o", LIB + ".tmp", "-lcudart", "-lnccl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libperrk_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
