"""GPU: the deterministic mode (pgm_context_config.deterministic =
PGM_DETERMINISTIC_PLANES, DeviceExecutor(deterministic=True)) — SURVEY §8(e)
"Determinism option": every reduction is per-plane sequential partials
(the reference's deterministic Executor::dot_kernel with block = n_axis^2,
parallel.cpp:120-131) combined by the reference's pairwise fold
(parallel.cpp:33-46).  The result depends only on the vectors, so

* the initial residual norm beta0 equals the reference deterministic
  executor's bit for bit (same vector b, same partials, same fold), and
* a whole solve is bit-identical for W = 1, 2, 3, 4 z-slab ranks
  (test_parallel.cpp:137-157 for the reference's dots), while matching the
  reference within the parity tolerances."""
import threading

import numpy as np
import pytest

import paper_1906_04051_b200 as pg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _ranks(world, fn):
    grp = pg.LoopbackGroup(world) if world > 1 else None
    out, err = {}, {}

    def body(r):
        try:
            out[r] = fn(r, grp)
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise next(iter(err.values()))
    return [out[r] for r in range(world)]


def _solve(ne, world, cfg, defl=True):
    na = 2 * ne + 1

    def rank(r, grp):
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world,
                               loopback=grp, deterministic=True)
        A, b = ex.assemble_bratu(ne, 6.8, device=False)
        x = np.zeros(ex.n_own)
        if defl:
            d = pg.Deflator(pg.DeflationConfig(), ex)
            rep = pg.deflated_gmres(A, b, x, cfg, d, ex)
            return rep, x, d.rank(), d.mu()
        rep = pg.gmres_restarted(A, None, b, x, cfg, ex)
        return rep, x, 0, 0.0

    res = _ranks(world, rank)
    return res[0][0], np.concatenate([rr[1] for rr in res]), res[0][2], res[0][3]


def test_det_beta0_equals_reference_bitwise(cuda, golden):
    g = golden("cfg1_defl")  # reference, deterministic executor (block = n_axis^2)
    rep, x, _, _ = _solve(10, 1, pg.GmresConfig(m=30, rel_tol=1e-10))
    assert rep.beta0 == float(g["beta0"])  # bit for bit
    assert abs(rep.total_inner - int(g["total_inner"])) <= 1
    b0 = float(g["beta0"])
    n = min(len(rep.monitored), len(g["monitored"]))
    assert np.max(np.abs(rep.monitored[:n] - g["monitored"][:n])) <= 1e-10 * b0
    assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])


@pytest.mark.parametrize("defl", [True, False])
def test_det_bit_identical_for_any_rank_count(cuda, golden, defl):
    cfg = pg.GmresConfig(m=30, rel_tol=1e-10)
    base = _solve(10, 1, cfg, defl)
    for world in (2, 3, 4):
        rep, x, rk, mu = _solve(10, world, cfg, defl)
        assert rep.beta0 == base[0].beta0, world
        assert rep.total_inner == base[0].total_inner, world
        assert np.array_equal(rep.monitored, base[0].monitored), world
        assert np.array_equal(rep.explicit_residual, base[0].explicit_residual), world
        assert np.array_equal(x, base[1]), world
        assert rk == base[2] and mu == base[3], world
    g = golden("cfg1_defl" if defl else "cfg1_plain")
    assert abs(base[0].total_inner - int(g["total_inner"])) <= 1
    assert np.linalg.norm(base[1] - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])


def test_det_truncation_run_bit_identical(cuda, golden):
    """24 fixed GMRES(4) cycles at n_e = 10 with 4 truncations (the harvest,
    push_vector, T row/column and rotation reductions all deterministic)."""
    cfg = pg.GmresConfig(m=4, max_restarts=24, fixed_iterations=True)
    r1 = _solve(10, 1, cfg)
    r3 = _solve(10, 3, cfg)
    assert np.array_equal(r1[0].monitored, r3[0].monitored)
    assert np.array_equal(r1[1], r3[1])
    g = golden("ne10_m4_trunc")
    assert np.linalg.norm(r1[1] - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])
