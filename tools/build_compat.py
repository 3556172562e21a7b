"""Build tests/cpp/_build/newton_compat: the reference's own src/newton.cpp,
assembly.cpp, mesh.cpp, sparse.cpp and parallel.cpp compiled VERBATIM (read
in place from /root/reference/proj, never copied) against the drop-in headers
include/compat/dgmres/{gmres,deflation}.hpp, linked with
paper_1906_04051_b200/compat/dgmres_device.cpp and libpgmres.so instead of
the reference's gmres.cpp / deflation.cpp.  Runs here (where the reference
sources exist); the binary travels to the GPU box with the repo snapshot.

    python tools/build_compat.py
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("DGMRES_REF", "/root/reference/proj")
OUT = os.path.join(ROOT, "tests", "cpp", "_build")
EXE = os.path.join(OUT, "newton_compat")
LIBDIR = os.path.join(ROOT, "paper_1906_04051_b200", "_lib")
REF_SOURCES = ["newton", "assembly", "mesh", "sparse", "parallel"]
CXX = os.environ.get("CXX", "g++")
# compat first: "dgmres/gmres.hpp" and "dgmres/deflation.hpp" resolve to the
# drop-in, every other dgmres/ header to the reference's own
INCLUDES = ["-I", os.path.join(ROOT, "include", "compat"), "-I", os.path.join(REF, "include"),
            "-I", os.path.join(ROOT, "include")]
FLAGS = ["-std=c++20", "-O2", "-DNDEBUG", "-fPIC", "-Wall", "-Wno-unused-parameter"]


def build() -> str:
    if not os.path.isdir(os.path.join(REF, "src")):
        if os.path.exists(EXE):
            return EXE
        raise RuntimeError("reference sources absent and newton_compat not prebuilt")
    os.makedirs(OUT, exist_ok=True)
    objs = []
    srcs = [(os.path.join(REF, "src", s + ".cpp"), s) for s in REF_SOURCES]
    srcs += [(os.path.join(ROOT, "paper_1906_04051_b200", "compat", "dgmres_device.cpp"),
              "dgmres_device"),
             (os.path.join(ROOT, "tests", "cpp", "newton_compat_main.cpp"), "main")]
    for src, name in srcs:
        obj = os.path.join(OUT, name + ".o")
        subprocess.run([CXX, *FLAGS, *INCLUDES, "-c", src, "-o", obj], check=True)
        objs.append(obj)
    subprocess.run([CXX, "-o", EXE, *objs, "-L", LIBDIR, "-lpgmres", "-lpthread",
                    "-Wl,-rpath,$ORIGIN/../../../paper_1906_04051_b200/_lib"], check=True)
    return EXE


if __name__ == "__main__":
    print(build())
    sys.exit(0)
