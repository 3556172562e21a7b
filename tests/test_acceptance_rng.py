"""CPU: paper_1906_04051_b200.rng reproduces std::mt19937(11) +
std::uniform_real_distribution<double>(-1, 1) (acceptance.cpp:437-443) bit
for bit (compiled against this machine's libstdc++)."""
import os
import subprocess

import numpy as np

from paper_1906_04051_b200.rng import acceptance_vectors

SRC = r"""
#include <cstdio>
#include <random>
int main() {
  std::mt19937 rng(11);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int i = 0; i < 5000; ++i) {
    const double v = dist(rng), w = dist(rng);
    std::printf("%a %a\n", v, w);
  }
}
"""


def test_acceptance_vectors_match_libstdcxx(tmp_path):
    src = tmp_path / "rng.cpp"
    src.write_text(SRC)
    exe = str(tmp_path / "rng")
    subprocess.run(["g++", "-O2", "-o", exe, str(src)], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    ref = np.array([float.fromhex(t) for t in out]).reshape(-1, 2)
    v, w = acceptance_vectors(5000)
    assert np.array_equal(v, ref[:, 0]) and np.array_equal(w, ref[:, 1])
