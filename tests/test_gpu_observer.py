"""GPU: the restart observer (RestartHook, gmres.hpp:94-113) through the C ABI
(pgm_set_restart_observer / pgm_restart_basis / pgm_restart_hessenberg).

* After every cycle the hook sees the cycle's basis and unrotated Hessenberg
  matrix: V^T V = I and the Arnoldi relation A v_j = sum_i h_ij v_i hold on
  the device's data (DCGS2 default and the CGS2 step).
* Criterion 8 of the reference's acceptance suite (acceptance.cpp:66-122,
  400-422): the deflation basis audited after every restart of the benchmark
  protocol (GMRES(50), 100 fixed restarts, n_e in {8, 15, 25}):
  ||U^T U - I||_max < 1e-10, ||T - U^T (A U)||_max / ||T||_max < 1e-10, rank <= 20.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_1906_04051_b200 as pg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _scipy(A):
    return sp.csr_matrix((A.values, A.col_idx.astype(np.int64), A.row_ptr.astype(np.int64)),
                         shape=(A.n, A.n))


@pytest.mark.parametrize("variant", ["dcgs2", "cgs2"])
def test_observer_sees_arnoldi_basis(torch_cuda, ref, monkeypatch, variant):
    monkeypatch.setenv("PGMRES_DCGS2", "1" if variant == "dcgs2" else "0")
    Ar, b = ref.first_newton_system(10)
    S = _scipy(Ar)
    A = pg.CsrMatrix(Ar.n, Ar.row_ptr, Ar.col_idx, Ar.values)
    ex = pg.DeviceExecutor()
    seen = []

    def hook(ctx):
        k = ctx.steps
        V = np.stack([ctx.ws.basis(j) for j in range(k)], axis=1)
        H = np.array([[ctx.ws.hess(i, j) for j in range(k - 1)] for i in range(k)])
        ortho = np.abs(V.T @ V - np.eye(k)).max()
        arn = np.abs(S @ V[:, : k - 1] - V @ H).max() / np.abs(H).max()
        seen.append((ctx.restart, k, ortho, arn))

    x = np.zeros(A.n)
    rep = pg.gmres_restarted(A, None, b, x, pg.GmresConfig(m=30, max_restarts=3,
                                                          fixed_iterations=True), ex, hook=hook)
    assert [s[0] for s in seen] == [0, 1, 2] and all(s[1] == 30 for s in seen)
    assert max(s[2] for s in seen) < 1e-12, seen
    assert max(s[3] for s in seen) < 1e-12, seen
    # the observer does not perturb the solve
    x2 = np.zeros(A.n)
    rep2 = pg.gmres_restarted(A, None, b, x2, pg.GmresConfig(m=30, max_restarts=3,
                                                            fixed_iterations=True), ex)
    assert np.array_equal(rep.monitored, rep2.monitored) and np.array_equal(x, x2)


def test_observer_exception_stops_solve(torch_cuda, ref):
    Ar, b = ref.first_newton_system(4)
    A = pg.CsrMatrix(Ar.n, Ar.row_ptr, Ar.col_idx, Ar.values)
    ex = pg.DeviceExecutor()

    def hook(ctx):
        if ctx.restart == 1:
            raise KeyError("audit failed")

    with pytest.raises(KeyError):
        pg.gmres_restarted(A, None, b, np.zeros(A.n),
                           pg.GmresConfig(m=5, max_restarts=4, fixed_iterations=True), ex,
                           hook=hook)
    # the context stays usable
    x = np.zeros(A.n)
    rep = pg.gmres_restarted(A, None, b, x, pg.GmresConfig(m=5, max_restarts=4,
                                                          fixed_iterations=True), ex)
    assert rep.restarts == 4


@pytest.mark.parametrize("ne", [8, 15, 25])
def test_criterion8_deflation_audit(torch_cuda, ref, ne):
    Ar, b = ref.first_newton_system(ne)
    S = _scipy(Ar)
    A = pg.CsrMatrix(Ar.n, Ar.row_ptr, Ar.col_idx, Ar.values)
    ex = pg.DeviceExecutor()
    d = pg.Deflator(pg.DeflationConfig(r_max=20))
    audit = dict(ortho=0.0, tmatch=0.0, rank=0, calls=0)

    def hook(ctx):
        audit["calls"] += 1
        r = d.rank()
        audit["rank"] = max(audit["rank"], r)
        if r == 0:
            return
        U = d.basis_matrix()
        audit["ortho"] = max(audit["ortho"], np.abs(U.T @ U - np.eye(r)).max())
        T = d.T_block()
        scale = max(np.abs(T).max(), 1e-300)
        audit["tmatch"] = max(audit["tmatch"], np.abs(T - U.T @ (S @ U)).max() / scale)

    x = np.zeros(A.n)
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=50, max_restarts=100,
                                                    fixed_iterations=True), d, ex,
                            observer=hook)
    assert rep.restarts == 100 and audit["calls"] == 100
    assert audit["ortho"] < 1e-10, audit
    assert audit["tmatch"] < 1e-10, audit
    assert audit["rank"] <= 20, audit
