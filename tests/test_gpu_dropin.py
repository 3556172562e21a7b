"""GPU: the C++ drop-in header (include/pgmres/dgmres.hpp) used the way the
reference's Newton driver calls deflated_gmres (newton.cpp:60-63), compiled
with g++ against libpgmres.so, must reproduce the reference's cfg1 solve."""
import os
import subprocess

import pytest

from paper_1906_04051_b200.build import LIBDIR, ROOT, build_library

pytestmark = pytest.mark.gpu


def test_cpp_dropin_cfg1(tmp_path, golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    build_library()
    exe = str(tmp_path / "dropin")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L", LIBDIR,
                    "-lpgmres", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    out = subprocess.run([exe, "10", "30"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    restarts, inner, rank, frel, mu, xn = out.stdout.split()
    g = golden("cfg1_defl")
    assert int(restarts) == int(g["restarts"]) and int(inner) == int(g["total_inner"])
    assert int(rank) == int(g["rank"])
    assert float(mu) == pytest.approx(float(g["mu"]), rel=1e-8)
    import numpy as np

    assert float(xn) == pytest.approx(float(np.linalg.norm(g["x"])), rel=1e-9)
