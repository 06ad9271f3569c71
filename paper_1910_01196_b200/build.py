"""Build the CUDA extension in-tree: paper_1910_01196_b200/liblocload_b200.so.

Plain nvcc, sm_100a only (no PTX fallback, no other arch), -lineinfo so ncu's
source page maps to the kernels.  The .so is git-ignored and travels to the
GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblocload_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

PER_FILE = {}

SOURCES = ["capi.cu", "permute.cu", "assign.cu", "shard.cu", "augment.cu", "exchange.cu",
           "loader.cu", "train.cu", "store.cu", "host/locload_api.cpp",
           "host/pipeline_api.cpp"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2,-Wall,-ffp-contract=off", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(d, f) for d in (CSRC, os.path.join(CSRC, "host"))
            for f in os.listdir(d) if os.path.isfile(os.path.join(d, f))]
    inc = os.path.join(ROOT, "include")
    for d, _, fs in os.walk(inc):
        deps += [os.path.join(d, f) for f in fs]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), lib=None) -> str:
    global LIB
    if lib is not None:  # variant builds for A/B measurements
        LIB = lib
        force = True
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    logs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src).rsplit(".", 1)[0] + ".o")
        cmd = [NVCC, *FLAGS, *PER_FILE.get(src, []), *extra, "-c", os.path.join(CSRC, src), "-o",
               obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-lnccl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
