"""CPU: the single-thread dense routines the device runs at restart time
(csrc/dense.cuh: LU inverse, Householder-Hessenberg + shifted complex QR eigenvalues, dominant eigenvector
for Deflator::truncate) against numpy/LAPACK."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest
from scipy.optimize import linear_sum_assignment

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dense(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("dense") / "dense_h.so")
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-o", so,
                    os.path.join(ROOT, "tests", "dense_harness.cpp")], check=True)
    L = C.CDLL(so)
    P = np.ctypeslib.ndpointer(np.float64, flags="C")
    L.h_dominant_eigvec.argtypes = [P, C.c_int, P]
    L.h_eigvals.argtypes = [P, C.c_int, P, P]
    L.h_invert.argtypes = [P, C.c_int, P]
    return L


def _f(A):
    return np.asfortranarray(A).ravel(order="F").copy()


def test_eigenvalues_match_lapack(dense):
    rng = np.random.default_rng(0)
    for trial in range(600):
        n = int(rng.integers(1, 24))
        A = rng.standard_normal((n, n))
        if trial % 3 == 1:
            A = A + A.T
        wr, wi = np.zeros(n), np.zeros(n)
        assert dense.h_eigvals(_f(A), n, wr, wi) == 0
        ev = wr + 1j * wi
        ref = np.linalg.eigvals(A)
        # pair the two spectra optimally (a sort would split conjugate pairs
        # whose real parts differ in the last bit)
        rows, cols = linear_sum_assignment(np.abs(ev[:, None] - ref[None, :]))
        assert np.max(np.abs(ev[rows] - ref[cols])) <= 1e-11 * max(1.0, np.abs(ref).max())


def test_dominant_eigenvector(dense):
    rng = np.random.default_rng(1)
    for _ in range(400):
        n = int(rng.integers(2, 22))
        A = rng.standard_normal((n, n))
        A = A + A.T + 1e-9 * rng.standard_normal((n, n))  # T is symmetric up to roundoff
        vals, vecs = np.linalg.eig(A)
        s = np.sort(np.abs(vals))
        if s[-1] - s[-2] < 1e-6 * s[-1]:
            continue
        v = np.zeros(n)
        assert dense.h_dominant_eigvec(_f(A), n, v) == 0
        ref = vecs[:, np.argmax(np.abs(vals))].real
        v, ref = v / np.linalg.norm(v), ref / np.linalg.norm(ref)
        assert min(np.linalg.norm(v - ref), np.linalg.norm(v + ref)) < 1e-10


def test_truncation_fixture_vectors(dense):
    # deflation.cpp test vectors: diag(1,2,3) -> dominant e3 (test_deflation.cpp:55-75)
    v = np.zeros(3)
    dense.h_dominant_eigvec(_f(np.diag([1.0, 2.0, 3.0])), 3, v)
    assert abs(abs(v[2]) - 1.0) < 1e-14 and np.abs(v[:2]).max() < 1e-14


def test_invert(dense):
    rng = np.random.default_rng(2)
    for _ in range(200):
        n = int(rng.integers(1, 22))
        A = rng.standard_normal((n, n)) + n * np.eye(n)
        inv = np.zeros(n * n)
        dense.h_invert(_f(A), n, inv)
        assert np.abs(inv.reshape(n, n, order="F") @ A - np.eye(n)).max() < 1e-12
