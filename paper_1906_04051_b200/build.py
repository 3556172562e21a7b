"""In-tree build of libpgmres.so (nvcc, sm_100a).  No JIT cache: the .so lives
next to the sources so it travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libpgmres.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h"))
                  + [os.path.join(ROOT, "include", "pgmres.h")])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, *FLAGS, "-o", tmp, os.path.join(CSRC, "pgmres.cu"), "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-8000:])
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
        f.write(res.stderr)
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines: list[str]) -> str:
    """A tuning variant (e.g. -DPGM_TILE=256) at _lib/variants/libpgmres_<name>.so,
    selected at run time with PGMRES_LIB=<path> (paper_1906_04051_b200/_capi.py)."""
    out = os.path.join(LIBDIR, "variants", f"libpgmres_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *ARCH, *FLAGS, *defines, "-o", out, os.path.join(CSRC, "pgmres.cu"), "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stderr[-8000:])
    with open(out + ".ptxas.log", "w") as f:
        f.write(res.stderr)
    return out


if __name__ == "__main__":
    import sys

    if len(sys.argv) > 2 and sys.argv[1] == "variant":
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        print(build_library(force=True))
