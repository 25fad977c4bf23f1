"""Build libgcb200.so in-tree with nvcc for sm_100a.

``python -m paper_1810_08429_b200.build_native`` (or ``__graft_entry__.build``)
compiles every ``csrc/*.cu`` into ``paper_1810_08429_b200/libgcb200.so``.
The library is a plain C-ABI shared object (``include/gcb200.h``); it links
the CUDA runtime statically and has no torch dependency.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgcb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=default", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-ldl"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith(".cu"))


def _deps():
    dep = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC)
                       if f.endswith(".cuh")]
    dep.append(os.path.join(ROOT, "include", "gcb200.h"))
    return dep


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build(force=False, verbose=False, extra=()):
    if not force and up_to_date():
        return LIB
    cmd = [NVCC] + ARCH + FLAGS + list(extra) + sources() + ["-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose and res.stderr:
        print(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else [])
    print(LIB)
