"""The reference acceptance suite's random vectors (acceptance.cpp:437-443):
std::mt19937 rng(11); std::uniform_real_distribution<double> dist(-1, 1);
v[i] = dist(rng); w[i] = dist(rng) — reproduced bit for bit with numpy's
MT19937 (legacy init_genrand seeding = std::mt19937's) and libstdc++'s
generate_canonical<double, 53> (two 32-bit draws, low word first) followed
by (b - a) * u + a.  Input generation for the SpMV microbenchmark (SURVEY
§8(d)); checked against libstdc++ in tests/test_acceptance_rng.py."""
from __future__ import annotations

import numpy as np


def mt19937_uniform(count: int, seed: int = 11, a: float = -1.0, b: float = 1.0) -> np.ndarray:
    bg = np.random.MT19937(0)
    bg._legacy_seeding(seed)
    raw = bg.random_raw(2 * count).astype(np.float64)
    s = raw[0::2] + raw[1::2] * 4294967296.0  # generate_canonical: sum += g * tmp (double)
    u = s / 18446744073709551616.0
    u = np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)
    return (b - a) * u + a


def acceptance_vectors(n: int, seed: int = 11):
    """(v, w) of acceptance.cpp:437-443 (draws interleaved v0, w0, v1, w1, ...)."""
    vals = mt19937_uniform(2 * n, seed)
    return vals[0::2].copy(), vals[1::2].copy()
