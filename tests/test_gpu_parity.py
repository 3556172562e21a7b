"""GPU parity: libpgmres (through the C ABI) against the reference.

Tolerances (north star): same iteration count +-1, residual
history within 1e-10 * beta0, solution within 1e-8 relative; SpMV bit-exact
(ascending-column accumulation, no FMA contraction, sparse.cpp:9-19)."""
import numpy as np
import pytest

import paper_1906_04051_b200 as pg

pytestmark = pytest.mark.gpu

HIST_TOL = 1e-10  # relative to beta0
X_TOL = 1e-8


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _csr(R, ne):
    A, b = R.first_newton_system(ne)
    return pg.CsrMatrix(A.n, A.row_ptr, A.col_idx, A.values), A, b


def _compare(rep, g, x, x_ref=None, total_tol=1):
    b0 = float(g["beta0"])
    assert rep.beta0 == pytest.approx(b0, rel=1e-12)
    assert abs(rep.total_inner - int(g["total_inner"])) <= total_tol
    n = min(len(rep.monitored), len(g["monitored"]))
    assert np.max(np.abs(rep.monitored[:n] - g["monitored"][:n])) <= HIST_TOL * b0
    k = min(len(rep.explicit_residual), len(g["explicit_residual"]))
    assert np.max(np.abs(rep.explicit_residual[:k] - g["explicit_residual"][:k])) <= HIST_TOL * b0
    if x_ref is not None:
        assert np.linalg.norm(x - x_ref) <= X_TOL * np.linalg.norm(x_ref)


# ---------------------------------------------------------------------------
# SpMV (sparse.cpp:9-19, Executor::spmv parallel.cpp:230-277)

def test_spmv_bitexact_bratu(torch_cuda, ref):
    for ne in (1, 2, 5, 10):
        A, Ar, _ = _csr(ref, ne)
        ex = pg.DeviceExecutor()
        x = np.random.default_rng(ne).uniform(-1, 1, A.n)
        y = ex.spmv(A, x)
        assert np.array_equal(y, ref.spmv(Ar, x)), ne


def test_spmv_bitexact_irregular(torch_cuda, ref):
    # empty rows, a dense row, long and short rows, unsorted-by-length tiles
    rng = np.random.default_rng(5)
    n = 3000
    lens = rng.integers(0, 40, n)
    lens[7] = 0
    lens[100] = n
    lens[2000:2600] = 1
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]).astype(np.uint32)
    va = rng.standard_normal(rp[-1])
    A = pg.CsrMatrix(n, rp, ci, va)
    x = rng.standard_normal(n)
    ex = pg.DeviceExecutor()
    from oracle.refbind import Csr
    assert np.array_equal(ex.spmv(A, x), ref.spmv(Csr(n, rp, ci, va), x))


def test_spmv_bitexact_wide_gaps_32bit_columns(torch_cuda, ref):
    """Column gaps >= 65536 force the 32-bit column layout (the 16-bit delta
    layout is used otherwise); both must give the reference's bits."""
    rng = np.random.default_rng(11)
    n = 70000
    lens = rng.integers(1, 6, n)
    rp = np.zeros(n + 1, np.uint32)
    rp[1:] = np.cumsum(lens)
    cols = []
    for i, l in enumerate(lens):
        c = {i, 0, n - 1} if i % 97 == 0 else {i}
        while len(c) < max(l, len(c)):
            c.add(int(rng.integers(0, n)))
        cols.append(np.array(sorted(c), np.uint32))
    lens = np.array([len(c) for c in cols])
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate(cols).astype(np.uint32)
    va = rng.standard_normal(rp[-1])
    A = pg.CsrMatrix(n, rp, ci, va)
    x = rng.standard_normal(n)
    ex = pg.DeviceExecutor()
    from oracle.refbind import Csr
    assert np.array_equal(ex.spmv(A, x), ref.spmv(Csr(n, rp, ci, va), x))


def test_spmv_device_pointers(torch_cuda, ref):
    torch = torch_cuda
    A, Ar, _ = _csr(ref, 4)
    ex = pg.DeviceExecutor()
    dA = ex.upload(A)
    x = np.random.default_rng(3).uniform(-1, 1, A.n)
    y = ex.spmv(dA, torch.tensor(x, device="cuda"))
    assert np.array_equal(y.cpu().numpy(), ref.spmv(Ar, x))
    # update_values (Newton reuses the pattern, assembly.cpp:253)
    dA.update_values(2.0 * A.values)
    assert np.array_equal(ex.spmv(dA, x), 2.0 * ref.spmv(Ar, x))


# ---------------------------------------------------------------------------
# The hot path: deflated_gmres / gmres_restarted

def test_cfg1_deflated(torch_cuda, ref, golden):
    A, _, b = _csr(ref, 10)
    g = golden("cfg1_defl")
    ex = pg.DeviceExecutor()
    d = pg.Deflator()
    x = np.zeros(A.n)
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), d, ex)
    assert rep.converged and not rep.breakdown
    assert rep.restarts == int(g["restarts"])
    _compare(rep, g, x, g["x"])
    assert d.rank() == int(g["rank"])
    assert d.mu() == pytest.approx(float(g["mu"]), rel=1e-8)
    h = d.history()
    assert [r.r for r in h] == list(g["hist_r"])
    assert np.allclose([r.smallest_ritz for r in h], g["hist_theta"], rtol=1e-7)
    # the last harvested Ritz vector is converged to inv_power_tol = 1e-10 ||H||
    # (deflation.cpp:46), so its T row/column agree to ~1e-7, the rest to 1e-12
    assert np.abs(d.T_block() - g["T"]).max() <= 1e-6 * np.abs(g["T"]).max()


def test_cfg1_plain(torch_cuda, ref, golden):
    A, _, b = _csr(ref, 10)
    g = golden("cfg1_plain")
    ex = pg.DeviceExecutor()
    x = np.zeros(A.n)
    rep = pg.gmres_restarted(A, None, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), ex)
    assert rep.converged and rep.restarts == int(g["restarts"])
    _compare(rep, g, x, g["x"])


def test_truncation_run_matches_reference(torch_cuda, ref, golden):
    A, _, b = _csr(ref, 10)
    g = golden("ne10_m4_trunc")
    ex = pg.DeviceExecutor()
    d = pg.Deflator()
    x = np.zeros(A.n)
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=4, max_restarts=24, fixed_iterations=True),
                            d, ex)
    assert rep.restarts == 24 and rep.total_inner == 96 and not rep.converged
    _compare(rep, g, x, g["x"], total_tol=0)
    assert [r.r for r in d.history()] == list(g["hist_r"])
    assert np.abs(d.T_block() - g["T"]).max() <= 1e-8 * np.abs(g["T"]).max()
    U = d.basis_matrix()
    assert np.abs(U.T @ U - np.eye(d.rank())).max() < 1e-10
    AU = np.stack([ex.spmv(A, U[:, j]) for j in range(d.rank())], axis=1)
    T = d.T_block()
    assert np.abs(T - U.T @ AU).max() < 1e-10 * np.abs(T).max()


def test_fixed_run_to_rounding_floor(torch_cuda, ref, golden):
    A, _, b = _csr(ref, 4)
    g = golden("ne4_fixed_trunc")
    ex = pg.DeviceExecutor()
    d = pg.Deflator()
    x = np.zeros(A.n)
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=10, max_restarts=26, fixed_iterations=True),
                            d, ex)
    assert rep.restarts == 26 and rep.total_inner == 260
    b0 = float(g["beta0"])
    assert np.max(np.abs(rep.explicit_residual - g["explicit_residual"])) <= HIST_TOL * b0
    assert d.rank() <= 20
    assert np.linalg.norm(x - g["x"]) <= X_TOL * np.linalg.norm(g["x"])


def test_dense_lu_equivalence(torch_cuda, golden):
    # criterion 4 (acceptance.cpp:214-261): n_e = 2, plain and deflated vs dense LU
    s = golden("ne2_system")
    n = s["rhs"].size
    A = pg.CsrMatrix(n, s["row_ptr"], s["col_idx"], s["values"])
    dense = np.zeros((n, n))
    for i in range(n):
        for k in range(s["row_ptr"][i], s["row_ptr"][i + 1]):
            dense[i, s["col_idx"][k]] = s["values"][k]
    xd = np.linalg.solve(dense, s["rhs"])
    ex = pg.DeviceExecutor()
    cfg = pg.GmresConfig(m=50, max_restarts=100, rel_tol=1e-12)
    x1 = np.zeros(n)
    pg.gmres_restarted(A, None, s["rhs"], x1, cfg, ex)
    x2 = np.zeros(n)
    pg.deflated_gmres(A, s["rhs"], x2, cfg, pg.Deflator(pg.DeflationConfig(r_max=20)), ex)
    assert np.linalg.norm(x1 - xd) <= 1e-10 * np.linalg.norm(xd)
    assert np.linalg.norm(x2 - xd) <= 1e-10 * np.linalg.norm(xd)


@pytest.mark.parametrize("variant", ["dcgs2", "cgs2"])
def test_finite_termination(torch_cuda, golden, ref, monkeypatch, variant):
    # test_gmres.cpp:232-254: one restart of length >= 45 free DOF exhausts the
    # space (the reference uses m = 125; the device bounds m by MAX_M = 112)
    monkeypatch.setenv("PGMRES_DCGS2", "1" if variant == "dcgs2" else "0")
    s = golden("ne2_system")
    n = s["rhs"].size
    A = pg.CsrMatrix(n, s["row_ptr"], s["col_idx"], s["values"])
    ex = pg.DeviceExecutor()
    x = np.zeros(n)
    cfg = pg.GmresConfig(m=112, max_restarts=1, rel_tol=1e-12)
    rep = pg.gmres_restarted(A, None, s["rhs"], x, cfg, ex)
    Ar = ref.Csr(n, s["row_ptr"], s["col_idx"], s["values"])
    r = ref.solve(Ar, s["rhs"], m=112, max_restarts=1, rel_tol=1e-12, deflation=False)
    assert rep.converged == r.converged and rep.breakdown == r.breakdown
    assert abs(rep.total_inner - r.total_inner) <= 1
    assert np.linalg.norm(x - r.x) <= X_TOL * np.linalg.norm(r.x)


def test_restart_length_bound(torch_cuda, golden):
    # every device path keeps a cycle's Hessenberg column in shared memory:
    # m > MAX_M is refused (PGM_EINVAL -> ValueError), never silently overrun
    s = golden("ne2_system")
    n = s["rhs"].size
    A = pg.CsrMatrix(n, s["row_ptr"], s["col_idx"], s["values"])
    ex = pg.DeviceExecutor()
    for defl in (None, pg.Deflator()):
        with pytest.raises(ValueError, match="restart length"):
            x = np.zeros(n)
            if defl is None:
                pg.gmres_restarted(A, None, s["rhs"], x, pg.GmresConfig(m=113), ex)
            else:
                pg.deflated_gmres(A, s["rhs"], x, pg.GmresConfig(m=113), defl, ex)


EXHAUST = [(6, 50, 1.0), (9, 40, 1e3), (5, 64, 1e-3), (12, 100, 1.0), (17, 300, 2.5)]


@pytest.mark.parametrize("variant", ["dcgs2", "cgs2"])
@pytest.mark.parametrize("fixed", [False, True])
def test_krylov_exhaustion_breakdown(torch_cuda, ref, monkeypatch, variant, fixed):
    """Exact Krylov exhaustion: diag(d) with k distinct eigenvalues and b
    spanning k eigenvectors -> h_{k,k-1} at rounding level after k steps; the
    lucky-breakdown exit (gmres.cpp:173-176, 189-192) must fire at the same
    step as the reference, in tolerance and fixed-iteration mode, with the
    same x."""
    monkeypatch.setenv("PGMRES_DCGS2", "1" if variant == "dcgs2" else "0")
    for k, n, scale in EXHAUST:
        d = np.tile(np.arange(1, k + 1, dtype=float) * scale, n // k + 1)[:n]
        b = np.ones(n)
        Ar = ref.diag_csr(d)
        r = ref.solve(Ar, b, m=30, max_restarts=3, rel_tol=1e-14, fixed_iterations=fixed,
                      deflation=False)
        assert r.breakdown and r.total_inner == k
        for defl in (False, True):
            ex = pg.DeviceExecutor()
            A = pg.CsrMatrix(n, Ar.row_ptr, Ar.col_idx, Ar.values)
            x = np.zeros(n)
            cfg = pg.GmresConfig(m=30, max_restarts=3, rel_tol=1e-14, fixed_iterations=fixed)
            if defl:
                rep = pg.deflated_gmres(A, b, x, cfg, pg.Deflator(), ex)
                rr = ref.solve(Ar, b, m=30, max_restarts=3, rel_tol=1e-14,
                               fixed_iterations=fixed, deflation=True)
            else:
                rep = pg.gmres_restarted(A, None, b, x, cfg, ex)
                rr = r
            assert rep.breakdown == rr.breakdown, (k, defl)
            assert rep.converged == rr.converged, (k, defl)
            assert rep.total_inner == rr.total_inner and rep.restarts == rr.restarts, (k, defl)
            assert np.linalg.norm(x - rr.x) <= X_TOL * np.linalg.norm(rr.x), (k, defl)
            assert np.max(np.abs(rep.monitored - rr.monitored)) <= HIST_TOL * rr.beta0


def test_crit10_spectral_action(torch_cuda, golden):
    # acceptance.cpp:539-595 on diag(1..50)
    g = golden("crit10_diag")
    n = 50
    A = pg.CsrMatrix(n, np.arange(n + 1, dtype=np.uint32), np.arange(n, dtype=np.uint32),
                     np.arange(1, n + 1, dtype=np.float64))
    ex = pg.DeviceExecutor()
    d = pg.Deflator(pg.DeflationConfig(r_max=20))
    x = np.zeros(n)
    pg.deflated_gmres(A, np.full(n, 1 / np.sqrt(n)), x,
                      pg.GmresConfig(m=8, max_restarts=5, fixed_iterations=True), d, ex)
    assert d.rank() == 5 and d.mu() == pytest.approx(float(g["mu"]), rel=1e-9)
    bm = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        bm[:, j] = np.arange(1, n + 1) * d.apply(e)
    ev = np.linalg.eigvals(bm)
    mu = d.mu()
    assert np.sum(np.abs(ev.real - mu) / mu < 0.05) >= 5
    assert ev.real.min() > 5.5 and np.abs(ev.imag).max() < 1e-8
    assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])


def test_crit3_midflight(torch_cuda, ref, golden):
    A, _, b = _csr(ref, 25)
    g = golden("crit3_ne25")
    ex = pg.DeviceExecutor()
    cfg = pg.GmresConfig(m=50, max_restarts=3, fixed_iterations=True)
    x = np.zeros(A.n)
    rd = pg.deflated_gmres(A, b, x, cfg, pg.Deflator(), ex)
    x2 = np.zeros(A.n)
    rp = pg.gmres_restarted(A, None, b, x2, cfg, ex)
    b0 = float(g["beta0"])
    assert np.max(np.abs(rd.explicit_residual - g["defl_explicit"])) <= HIST_TOL * b0
    assert np.max(np.abs(rp.explicit_residual - g["plain_explicit"])) <= HIST_TOL * b0
    assert np.max(np.abs(rd.monitored - g["defl_monitored"])) <= HIST_TOL * b0


def _check_x_full(xh, x_ref):
    # north star: final solution within 1e-8 relative, no slack
    assert np.linalg.norm(xh - x_ref) <= X_TOL * np.linalg.norm(x_ref)


def _check_hist(rep, g, p):
    b0 = float(g[p + "beta0"])
    assert rep.beta0 == pytest.approx(b0, rel=1e-12)
    assert rep.converged == bool(g[p + "converged"])
    assert rep.breakdown == bool(g[p + "breakdown"])
    assert abs(rep.total_inner - int(g[p + "total_inner"])) <= 1
    assert abs(rep.restarts - int(g[p + "restarts"])) <= 1
    n = min(len(rep.monitored), len(g[p + "monitored"]))
    assert np.max(np.abs(rep.monitored[:n] - g[p + "monitored"][:n])) <= HIST_TOL * b0
    k = min(len(rep.explicit_residual), len(g[p + "explicit"]))
    assert np.max(np.abs(rep.explicit_residual[:k] - g[p + "explicit"][:k])) <= HIST_TOL * b0


def _plane_norms(x, ne):
    na = 2 * ne + 1
    return np.linalg.norm(x.reshape(na, na * na), axis=1)


@pytest.mark.slow
@pytest.mark.parametrize("defl", [True, False])
def test_cfg2_full_solution(torch_cuda, golden, defl):
    """BASELINE config 2: n_e = 50 (1,030,301 DOF), GMRES(50), tol 1e-10,
    deflated (reference: 9 restarts / 418 inner) and undeflated (41 / 2050);
    the FULL solution vector within 1e-8 of the reference's
    (tests/golden/make_golden_r2.py), histories within 1e-10 * beta0."""
    torch = torch_cuda
    g = golden("cfg2_full")
    p = "defl_" if defl else "plain_"
    ex = pg.DeviceExecutor()
    A, b = ex.assemble_bratu(50, 6.8, device=True)
    x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
    cfg = pg.GmresConfig(m=50, rel_tol=1e-10)
    if defl:
        d = pg.Deflator(pg.DeflationConfig(), ex)
        rep = pg.deflated_gmres(A, b, x, cfg, d, ex)
        assert d.rank() == int(g[p + "rank"])
        assert d.mu() == pytest.approx(float(g[p + "mu"]), rel=1e-6)
    else:
        rep = pg.gmres_restarted(A, None, b, x, cfg, ex)
    _check_hist(rep, g, p)
    _check_x_full(x.cpu().numpy(), g[p + "x"])


@pytest.mark.slow
@pytest.mark.parametrize("m", [20, 50, 100])
@pytest.mark.parametrize("defl", [True, False])
def test_sweep_ne31(torch_cuda, golden, m, defl):
    """BASELINE config 5's smallest mesh (n_e = 31, 250,047 DOF; "500^2") at
    every restart length and deflation on/off against the reference: counts,
    histories, x (every 4th entry) and the l2 norm of x on every node plane
    within 1e-8 relative."""
    torch = torch_cuda
    g = golden("sweep_ne31")
    p = f"m{m}_{'defl' if defl else 'plain'}_"
    ex = pg.DeviceExecutor()
    A, b = ex.assemble_bratu(31, 6.8, device=True)
    x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
    cfg = pg.GmresConfig(m=m, max_restarts=300, rel_tol=1e-10)
    if defl:
        d = pg.Deflator(pg.DeflationConfig(), ex)
        rep = pg.deflated_gmres(A, b, x, cfg, d, ex)
        assert d.rank() == int(g[p + "rank"])
    else:
        rep = pg.gmres_restarted(A, None, b, x, cfg, ex)
    _check_hist(rep, g, p)
    xh = x.cpu().numpy()
    _check_x_full(xh[::4], g[p + "x_stride4"])
    pn = _plane_norms(xh, 31)
    assert np.max(np.abs(pn - g[p + "x_planes"])) <= X_TOL * np.linalg.norm(g[p + "x_planes"])


# ---------------------------------------------------------------------------
# Unit-level ports of test_gmres.cpp / test_deflation.cpp

def _diag(vals):
    n = len(vals)
    return pg.CsrMatrix(n, np.arange(n + 1, dtype=np.uint32), np.arange(n, dtype=np.uint32),
                        np.asarray(vals, np.float64))


def test_identity_converges_at_first_step(torch_cuda):
    ex = pg.DeviceExecutor()
    b = np.array([1.0, -2.0, 3.0, 0.5, -0.25])
    x = np.zeros(5)
    rep = pg.gmres_restarted(_diag(np.ones(5)), None, b, x, pg.GmresConfig(m=5), ex)
    assert rep.converged and rep.breakdown and rep.total_inner == 1
    assert abs(rep.monitored[0]) < 1e-14
    assert np.allclose(x, b, atol=1e-14)


def test_scaled_identity_and_eigenvector_start(torch_cuda):
    ex = pg.DeviceExecutor()
    x = np.zeros(3)
    rep = pg.gmres_restarted(_diag([2.0, 2.0, 2.0]), None, np.array([4.0, 0, 0]), x,
                             pg.GmresConfig(), ex)
    assert rep.converged and abs(x[0] - 2.0) < 1e-15 and np.abs(x[1:]).max() < 1e-15
    ex2 = pg.DeviceExecutor()
    x = np.zeros(3)
    rep = pg.gmres_restarted(_diag([1.0, 2.0, 3.0]), None, np.array([1.0, 0, 0]), x,
                             pg.GmresConfig(), ex2)
    assert rep.breakdown and rep.converged and rep.total_inner == 1 and abs(x[0] - 1) < 1e-15


def test_plane_rotation(torch_cuda):
    # test_gmres.cpp:108-137: A = [[0,-1],[1,0]], b = e1 -> x = (0, -1)
    A = pg.CsrMatrix(2, np.array([0, 1, 2], np.uint32), np.array([1, 0], np.uint32),
                     np.array([-1.0, 1.0]))
    ex = pg.DeviceExecutor()
    x = np.zeros(2)
    rep = pg.gmres_restarted(A, None, np.array([1.0, 0.0]), x, pg.GmresConfig(m=2), ex)
    assert rep.monitored[0] == 1.0 and rep.monitored[1] == 0.0
    assert np.allclose(x, [0.0, -1.0], atol=1e-15)


def test_zero_rhs_and_errors(torch_cuda):
    ex = pg.DeviceExecutor()
    x = np.zeros(4)
    rep = pg.gmres_restarted(_diag(np.ones(4)), None, np.zeros(4), x, pg.GmresConfig(), ex)
    assert rep.converged and rep.total_inner == 0 and rep.restarts == 0
    with pytest.raises(ValueError):
        pg.gmres_restarted(_diag(np.ones(4)), None, np.ones(4), x, pg.GmresConfig(m=0), ex)
    bad = _diag([np.nan, 1.0])
    ex2 = pg.DeviceExecutor()
    with pytest.raises(pg.GmresError):
        pg.gmres_restarted(bad, None, np.ones(2), np.zeros(2), pg.GmresConfig(), ex2)
    with pytest.raises(ValueError):
        pg.Deflator(pg.DeflationConfig(r_max=0))
    with pytest.raises(ValueError):
        pg.Deflator(pg.DeflationConfig(r_max=5, drop=0))


def test_fixed_iteration_mode(torch_cuda):
    rng = np.random.default_rng(61)
    n = 8
    r = rng.standard_normal((n, n))
    a = r.T @ r + n * np.eye(n)
    rp = np.arange(0, n * n + 1, n, dtype=np.uint32)
    ci = np.tile(np.arange(n, dtype=np.uint32), n)
    A = pg.CsrMatrix(n, rp, ci, a.ravel())
    ex = pg.DeviceExecutor()
    x = np.zeros(n)
    rep = pg.gmres_restarted(A, None, rng.standard_normal(n), x,
                             pg.GmresConfig(m=2, max_restarts=7, fixed_iterations=True,
                                            rel_tol=1e-1), ex)
    assert rep.restarts == 7 and len(rep.explicit_residual) == 7 and rep.total_inner == 14
    assert not rep.converged


def test_deflator_truncation_exact(torch_cuda):
    # test_deflation.cpp:55-75
    ex = pg.DeviceExecutor()
    A = _diag([1.0, 2.0, 3.0])
    d = pg.Deflator()
    for i in range(3):
        e = np.zeros(3)
        e[i] = 1.0
        assert d.push_vector(e, A, ex)
    assert d.rank() == 3
    d.truncate()
    assert d.rank() == 2
    T = d.T_block()
    assert np.allclose(T, np.diag([1.0, 2.0]), atol=1e-14)
    U = d.basis_matrix()
    assert np.abs(U[2, :]).max() < 1e-14


def test_deflator_cap_and_span(torch_cuda):
    # test_deflation.cpp:77-104
    ex = pg.DeviceExecutor()
    A = _diag([1.0, 2.0, 3.0, 4.0, 5.0])
    d = pg.Deflator(pg.DeflationConfig(r_max=3))
    for i in range(4):
        e = np.zeros(5)
        e[i] = 1.0
        assert d.push_vector(e, A, ex)
    assert d.rank() == 3
    assert np.allclose(np.diag(d.T_block()), [1.0, 2.0, 3.0], atol=1e-12)
    ex2 = pg.DeviceExecutor()
    A3 = _diag([1.0, 2.0, 3.0])
    d2 = pg.Deflator()
    e0 = np.array([1.0, 0.0, 0.0])
    assert d2.push_vector(e0, A3, ex2)
    assert not d2.push_vector(e0, A3, ex2)
    assert d2.rank() == 1 and d2.skipped_updates() >= 1
    assert not d2.push_vector(np.zeros(3), A3, ex2)


def test_deflator_apply_dense_formula(torch_cuda):
    # test_deflation.cpp:103-142 (seed 77 style: random SPD, 4 random candidates)
    rng = np.random.default_rng(77)
    n, r = 30, 4
    gm = rng.standard_normal((n, n))
    a = gm.T @ gm + n * np.eye(n)
    A = pg.CsrMatrix(n, np.arange(0, n * n + 1, n, dtype=np.uint32),
                     np.tile(np.arange(n, dtype=np.uint32), n), a.ravel())
    ex = pg.DeviceExecutor()
    d = pg.Deflator()
    for j in range(r):
        assert d.push_vector(rng.standard_normal(n), A, ex)
    d.observe_ritz(123.5)
    U = d.basis_matrix()
    t = U.T @ a @ U
    minv = np.eye(n) + U @ (123.5 * np.linalg.inv(t) - np.eye(r)) @ U.T
    v = rng.standard_normal(n)
    assert np.abs(d.apply(v) - minv @ v).max() < 1e-11
    d.reset()
    assert d.rank() == 0 and d.mu() == 0.0 and d.history() == []
    assert np.array_equal(d.apply(v), v)


def test_deflator_exact_eigenvectors_to_mu(torch_cuda):
    # test_deflation.cpp:144-170
    ex = pg.DeviceExecutor()
    dvals = np.arange(1, 9, dtype=np.float64)
    A = _diag(dvals)
    d = pg.Deflator()
    for i in (1, 4):
        e = np.zeros(8)
        e[i] = 1.0
        assert d.push_vector(e, A, ex)
    d.observe_ritz(8.0)
    for i in (1, 4):
        e = np.zeros(8)
        e[i] = 1.0
        aw = dvals * d.apply(e)
        want = np.zeros(8)
        want[i] = 8.0
        assert np.abs(aw - want).max() < 1e-13
    e6 = np.zeros(8)
    e6[6] = 1.0
    assert np.abs(d.apply(e6) - e6).max() < 1e-13


def test_report_csv_round_trip(torch_cuda, ref):
    A, _, b = _csr(ref, 1)
    ex = pg.DeviceExecutor()
    x = np.zeros(A.n)
    rep = pg.gmres_restarted(A, None, b, x,
                             pg.GmresConfig(m=4, max_restarts=3, fixed_iterations=True), ex)
    lines = rep.write_csv().strip().split("\n")
    assert lines[0] == "restart,inner_step,monitored_residual,explicit_residual"
    closing = 0
    for i, line in enumerate(lines[1:]):
        r, k, mon, tail = line.split(",")
        assert float(mon) == rep.monitored[i]
        if tail:
            assert float(tail) == rep.explicit_residual[int(r)]
            closing += 1
    assert closing == len(rep.explicit_residual)


@pytest.mark.slow
def test_cfg3_deflated_full_size(torch_cuda, golden):
    """BASELINE config 3 on one B200: n_e = 125 (15,813,251 DOF, 991,266,025 nnz),
    GMRES(50) + deflation, tol 1e-10, assembled on the device (bit-identical to
    the reference assembly at u = 0).  The reference run (tests/golden/
    make_golden_large.py, 8 threads, 24 min) gives 24 restarts / 1181 inner
    with truncation active from restart 20; histories within 1e-10 * beta0,
    the solution (every 16th entry, per-plane norms) within 1e-8."""
    torch = torch_cuda
    g = golden("cfg3_defl")
    ex = pg.DeviceExecutor()
    A, b = ex.assemble_bratu(125, 6.8, device=True)
    d = pg.Deflator(pg.DeflationConfig(), ex)
    x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=50, rel_tol=1e-10), d, ex)
    assert rep.converged
    assert abs(rep.restarts - int(g["restarts"])) <= 1
    _compare(rep, g, None)
    xh = x.cpu().numpy()
    xn = float(g["x_norm"])
    assert abs(np.linalg.norm(xh) - xn) <= X_TOL * xn
    # the solution every 16th entry and its l2 norm on every node plane,
    # within the north star's 1e-8 (tests/golden/make_golden_r2.py cfg3)
    gx = golden("cfg3_x")
    assert int(gx["total_inner"]) == int(g["total_inner"])
    _check_x_full(xh[::16], gx["x_stride16"])
    pn = _plane_norms(xh, 125)
    assert np.max(np.abs(pn - gx["x_planes"])) <= X_TOL * np.linalg.norm(gx["x_planes"])
    assert d.rank() == int(g["rank"])
    hr = np.array([h.r for h in d.history()])
    k = min(len(hr), len(g["hist_r"]))
    assert np.array_equal(hr[:k], g["hist_r"][:k]), (hr, g["hist_r"])


@pytest.mark.parametrize("m,defl", [(20, True), (20, False), (100, True), (100, False)])
def test_restart_length_sweep_ne25(torch_cuda, golden, m, defl):
    """BASELINE config 5's restart sweep (m in {20, 50, 100}, deflation on and
    off; m = 50 is cfg2) on n_e = 25 against the reference
    (tests/golden/make_golden_sweep.py).  m = 100 runs the 8-warp pass-B
    kernels (more than 64 basis vectors)."""
    g = golden("sweep_ne25")
    key = f"m{m}_{'defl' if defl else 'plain'}"
    ex = pg.DeviceExecutor()
    A, b = ex.assemble_bratu(25, 6.8, device=True)
    x = torch_cuda.zeros(ex.n_own, dtype=torch_cuda.float64, device="cuda")
    cfg = pg.GmresConfig(m=m, max_restarts=200, rel_tol=1e-10)
    if defl:
        rep = pg.deflated_gmres(A, b, x, cfg, pg.Deflator(pg.DeflationConfig(), ex), ex)
    else:
        rep = pg.gmres_restarted(A, None, b, x, cfg, ex)
    b0 = float(g[key + "_beta0"])
    assert rep.converged
    assert abs(rep.total_inner - int(g[key + "_total_inner"])) <= 1
    n = min(len(rep.monitored), len(g[key + "_monitored"]))
    assert np.max(np.abs(rep.monitored[:n] - g[key + "_monitored"][:n])) <= HIST_TOL * b0
    xh = x.cpu().numpy()
    assert abs(np.linalg.norm(xh) - float(g[key + "_x_norm"])) <= X_TOL * float(g[key + "_x_norm"])
    assert np.linalg.norm(xh[::97] - g[key + "_x_sample"]) <= X_TOL * np.linalg.norm(
        g[key + "_x_sample"])


@pytest.mark.parametrize("variant", ["cgs2"])
def test_cgs2_path_still_matches(torch_cuda, ref, golden, monkeypatch, variant):
    """PGMRES_DCGS2=0 keeps the two-reduction CGS2 step (pass B + pass C) —
    the DCGS2 default's fallback (peer transport with a large restart length)."""
    monkeypatch.setenv("PGMRES_DCGS2", "0")
    A, _, b = _csr(ref, 10)
    g = golden("cfg1_defl")
    ex = pg.DeviceExecutor()
    d = pg.Deflator()
    x = np.zeros(A.n)
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), d, ex)
    assert rep.restarts == int(g["restarts"])
    _compare(rep, g, x, g["x"])
    gt = golden("ne10_m4_trunc")
    A2, _, b2 = _csr(ref, 10)
    d2 = pg.Deflator()
    x2 = np.zeros(A2.n)
    pg.deflated_gmres(A2, b2, x2, pg.GmresConfig(m=4, max_restarts=24, fixed_iterations=True), d2,
                      pg.DeviceExecutor())
    assert [h.r for h in d2.history()] == list(gt["hist_r"])


@pytest.mark.slow
def test_ne200_fixed_cycles_and_fit(torch_cuda, golden):
    """BASELINE config 5's largest mesh, n_e = 200 ("8000^2": 64,481,201 DOF,
    4,073,625,625 nnz — gaps exceed 16 bits, so the 32-bit column layout).
    (1) Deflated GMRES(20), 2 fixed cycles, against the reference run on the
    GPU box's host (tests/golden/make_golden_ne200.py): histories within
    1e-10 * beta0, x (every 64th entry) and per-plane norms within 1e-8.
    (2) BASELINE's largest restart length m = 100 fits in HBM next to the
    matrix (no resident CSR staging): 2 fixed deflated cycles, monitored and
    explicit residuals consistent at every cycle end."""
    import os

    torch = torch_cuda
    if not os.path.exists(os.path.join(os.path.dirname(__file__), "golden", "ne200_fixed.npz")):
        pytest.skip("ne200 golden not generated")
    g = golden("ne200_fixed")
    ex = pg.DeviceExecutor()
    A, b = ex.assemble_bratu(200, 6.8, device=True)
    dA = ex.upload(A)
    del A
    torch.cuda.empty_cache()
    info = dA.info()
    assert info["nnz"] == 4073625625
    assert info["device_bytes"] >= 12 * info["stored"]  # 32-bit column ids
    x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
    cfg = pg.GmresConfig(m=20, max_restarts=2, fixed_iterations=True)
    d = pg.Deflator(pg.DeflationConfig(), ex)
    rep = pg.deflated_gmres(dA, b, x, cfg, d, ex)
    b0 = float(g["beta0"])
    assert rep.beta0 == pytest.approx(b0, rel=1e-12)
    assert rep.total_inner == int(g["total_inner"]) and rep.restarts == int(g["restarts"])
    assert np.max(np.abs(rep.monitored - g["monitored"])) <= HIST_TOL * b0
    assert np.max(np.abs(rep.explicit_residual - g["explicit"])) <= HIST_TOL * b0
    assert d.rank() == int(g["rank"])
    xh = x.cpu().numpy()
    _check_x_full(xh[::64], g["x_stride64"])
    pn = _plane_norms(xh, 200)
    assert np.max(np.abs(pn - g["x_planes"])) <= X_TOL * np.linalg.norm(g["x_planes"])
    del xh
    # (2) m = 100
    x.zero_()
    rep = pg.deflated_gmres(dA, b, x, pg.GmresConfig(m=100, max_restarts=2, fixed_iterations=True),
                            pg.Deflator(pg.DeflationConfig(), ex), ex)
    assert rep.total_inner == 200 and np.all(np.isfinite(rep.explicit_residual))
    mon = np.asarray(rep.monitored)
    for c in range(2):
        assert abs(mon[100 * c + 99] - rep.explicit_residual[c]) <= 1e-6 * rep.beta0
    assert rep.explicit_residual[1] < rep.explicit_residual[0] < rep.beta0
