"""Build libmsd.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with
the repo snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmsd.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    s = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
    s += sorted(glob.glob(os.path.join(HERE, "csrc", "*.cpp")))
    return s


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
        sorted(glob.glob(os.path.join(HERE, "csrc", "*.h"))) + [os.path.join(ROOT, "include", "msd.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build libmsd.so (or libmsd_<variant>.so with extra -D defines, for A/B experiments)."""
    lib = LIB if not variant else os.path.join(HERE, f"libmsd_{variant}.so")
    if not force and not variant and up_to_date():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-cudart", "static", *[f"-D{d}" for d in defines], "-o", lib + ".tmp", *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd, cwd=HERE)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
