"""Build the in-tree C-ABI library (sm_100a) — `python -m paper_2603_10726_b200.build`."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "solid.cu"), os.path.join(PKG, "csrc", "solid_activator.cu")]
DEPS = SRC + sorted(os.path.join(PKG, "csrc", f) for f in os.listdir(os.path.join(PKG, "csrc"))
                    if f.endswith((".inc", ".cuh"))) + [os.path.join(ROOT, "include", "solid.h")]
LIB = os.path.join(PKG, "lib", "libsolid.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-diag-suppress", "186"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, counters: bool = False) -> str:
    """counters=True builds the profiling variant lib/libsolid_counters.so (-DSOLID_COUNTERS:
    per-round path counters, perturbs timing; load it with SOLID_LIB=...)."""
    lib = LIB.replace("libsolid.so", "libsolid_counters.so") if counters else LIB
    if not force and not counters and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-DSOLID_COUNTERS"] if counters else []),
           "-I", os.path.join(ROOT, "include"), "-o", tmp, *SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libsolid.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, counters="--counters" in sys.argv))
