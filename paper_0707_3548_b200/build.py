"""Build libtqr.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with gpurun)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
PHASES = os.environ.get("TQR_PHASES", "0") == "1"   # profiling variant with phase timers
# experiment variants (development only): extra -D flags and their own library name
VARIANT_DEFS = os.environ.get("TQR_VARIANT_DEFS", "").split()
VARIANT = os.environ.get("TQR_VARIANT", "")
LIB = os.path.join(HERE, f"libtqr_{VARIANT}.so" if VARIANT else ("libtqr_phases.so" if PHASES else "libtqr.so"))
SOURCES = ["tqr_exec.cu", "tqr_host.cpp", "tlu_exec.cu", "tlu_host.cpp"]
HEADERS = ["tqr_device.cuh", "tqr_internal.h", "tqr_sched.h", "tlu_internal.h", os.path.join("..", "..", "include", "tlu.h"), os.path.join("..", "..", "include", "tqr.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"] + (["-DTQR_PROFILE_PHASES"] if PHASES else []) + VARIANT_DEFS


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src + (f".{VARIANT}" if VARIANT else (".ph" if PHASES else "")) + ".o")
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs, "-lcudart"]
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
