"""CPU: the source-compatible drop-in (include/compat/dgmres) compiles the
reference's own src/newton.cpp, assembly.cpp, mesh.cpp, sparse.cpp and
parallel.cpp unchanged (syntax and semantic check with g++, no link, no GPU),
and the device implementation compiles against it.  Skipped where the
reference sources are absent (the GPU box); tests/test_gpu_compat.py runs the
linked binary there."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.environ.get("DGMRES_REF", "/root/reference/proj")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "src")), reason="reference sources absent")
@pytest.mark.parametrize("src", ["src/newton.cpp", "src/assembly.cpp", "src/parallel.cpp",
                                 "compat", "main"])
def test_reference_sources_compile_against_dropin(src):
    inc = ["-I", os.path.join(ROOT, "include", "compat"), "-I", os.path.join(REF, "include"),
           "-I", os.path.join(ROOT, "include")]
    path = {"compat": os.path.join(ROOT, "paper_1906_04051_b200", "compat", "dgmres_device.cpp"),
            "main": os.path.join(ROOT, "tests", "cpp", "newton_compat_main.cpp")}.get(
                src, os.path.join(REF, src))
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", *inc, path],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "src")), reason="reference sources absent")
def test_dropin_types_match_reference_layout():
    """GmresConfig / GmresReport / DeflationConfig of the drop-in have the
    reference's fields in the reference's order (designated initialisers of
    newton.hpp:18 compile, and the structs are layout-identical)."""
    code = r'''
#include "dgmres/deflation.hpp"
#include <cstddef>
static_assert(sizeof(dgmres::GmresConfig) == 32, "GmresConfig layout");
static_assert(offsetof(dgmres::GmresConfig, rel_tol) == 8, "rel_tol");
static_assert(offsetof(dgmres::GmresConfig, breakdown_scale) == 24, "breakdown_scale");
static_assert(offsetof(dgmres::DeflationConfig, accept_tol) == 8, "accept_tol");
dgmres::GmresConfig g{.m = 50, .max_restarts = 100, .rel_tol = 1e-10};
int main() { return g.m == 50 ? 0 : 1; }
'''
    inc = ["-I", os.path.join(ROOT, "include", "compat"), "-I", os.path.join(REF, "include"),
           "-I", os.path.join(ROOT, "include")]
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", *inc, "-"],
                       input=code, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
