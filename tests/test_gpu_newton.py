"""GPU parity of the device-resident Newton driver (pgm_newton_solve) against
the reference's newton_solve (newton.cpp:31-97) run through oracle/_ref.

Per-Newton-step tolerances: the linear solves carry the path's parity bar
(iteration count within a few, solution 1e-8 relative), so the Newton
iterates agree to ~1e-8 and the per-step records follow.  SURVEY.md §8(c):
even the reference's own executors differ by 2 inner iterations on the last,
hardest solve of the n_e = 8 run (95 vs 97), and at config 4 (n_e = 79)
its deterministic and non-deterministic executors differ by +1 / -2 on
steps 4 / 5; steps after the first get +-3 or 1.5 %.  Measured deltas
(B200): n_e = 8: 0 on every step (577 total, as the reference's sequential
executor); n_e = 79 (cfg4): 0, 0, +2, +4, -10."""
import numpy as np
import pytest

import paper_1906_04051_b200 as pg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _check_records(rep, g, n_steps):
    assert len(rep.iters) == n_steps
    inner = np.array([r.gmres_inner for r in rep.iters])
    # step 1 solves the same system as the reference: +-1 (north star).  Later
    # steps solve J(u_k) with u_k within ~1e-9 of the reference's, and their
    # late, near-stagnating GMRES runs are sensitive to rounding: the
    # reference's OWN deterministic vs non-deterministic executors give
    # 686/698/731/765/789 vs 686/698/731/766/787 at config 4
    # (profiles/r2_reference_newton79_spread.json); the device's DCGS2 step
    # 686/698/733/769/779.  Bound: +-3 or 1.5 %.
    assert abs(int(inner[0]) - int(g["inner"][0])) <= 1, (inner, g["inner"])
    tol = np.maximum(3, np.ceil(0.015 * g["inner"][:n_steps]))
    assert np.all(np.abs(inner - g["inner"][:n_steps]) <= tol), (inner, g["inner"])
    res = np.array([r.residual_norm for r in rep.iters])
    # ||R(u)||_2: relative 1e-6, floored at 1e-12 of the first (rounding floor of R)
    assert np.allclose(res, g["residual_norm"][:n_steps], rtol=1e-6,
                       atol=1e-12 * float(g["residual_norm"][0]))
    upd = np.array([r.update_inf for r in rep.iters])
    # ||delta||_inf: relative 1e-6 while the update is large, absolute at the end
    assert np.all(np.abs(upd - g["update_inf"][:n_steps]) <= 1e-6 * np.maximum(upd, 1e-3))


def test_newton_ne8_matches_reference(torch_cuda, golden):
    """Criterion 7 system (n_e = 8, lambda = 6.8, default NewtonConfig): the
    reference converges in 8 iterations to max u = 1.323002464567."""
    g = golden("newton_ne8")
    ex = pg.DeviceExecutor()
    u = np.zeros((2 * 8 + 1) ** 3)
    rep = pg.newton_solve(8, 6.8, u, pg.NewtonConfig(), ex)
    assert rep.converged
    _check_records(rep, g, len(g["inner"]))
    assert np.linalg.norm(u - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])
    assert abs(u.max() - 1.323002464567) < 1e-11
    assert rep.total_inner == sum(r.gmres_inner for r in rep.iters)
    csv = rep.write_csv()
    assert csv.splitlines()[0] == "iter,update_inf_norm,residual_2norm,gmres_restarts"
    assert len(csv.splitlines()) == 1 + len(rep.iters)


def test_newton_device_iterate_and_plain_gmres(torch_cuda, golden):
    """u as a CUDA tensor; use_deflation = False takes gmres_restarted(opA,
    nullptr) per step (newton.cpp:64-70) and still converges to the same u."""
    torch = torch_cuda
    g = golden("newton_ne8")
    ex = pg.DeviceExecutor()
    u = torch.zeros((2 * 8 + 1) ** 3, dtype=torch.float64, device="cuda")
    rep = pg.newton_solve(8, 6.8, u, pg.NewtonConfig(use_deflation=False), ex)
    assert rep.converged
    uh = u.cpu().numpy()
    assert np.linalg.norm(uh - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])


def test_newton_errors(torch_cuda):
    ex = pg.DeviceExecutor()
    u = np.zeros(27)
    with pytest.raises(ValueError, match="max_iters must be positive"):
        pg.newton_solve(1, 6.8, u, pg.NewtonConfig(max_iters=0), ex)


def test_newton_continuation_runs_stages(torch_cuda):
    """continuation: lambda ramps over continuation_steps stages (newton.cpp:36-42)."""
    ex = pg.DeviceExecutor()
    u = np.zeros((2 * 4 + 1) ** 3)
    rep = pg.newton_solve(4, 6.8, u, pg.NewtonConfig(continuation=True, continuation_steps=3),
                          ex)
    assert rep.converged
    lams = sorted({round(r.lam, 12) for r in rep.iters})
    assert lams == [round(6.8 * q / 3, 12) for q in (1, 2, 3)]


@pytest.mark.slow
def test_newton_cfg4_five_steps(torch_cuda, golden):
    """BASELINE config 4 on one B200: 5 Newton steps on n_e = 79 (4,019,679 DOF),
    deflated GMRES(50) to 1e-10 per step, against the reference's run
    (tests/golden/make_golden_large.py: 686/698/731/765/789 inner)."""
    torch = torch_cuda
    g = golden("newton79")
    ex = pg.DeviceExecutor()
    u = torch.zeros((2 * 79 + 1) ** 3, dtype=torch.float64, device="cuda")
    rep = pg.newton_solve(79, 6.8, u, pg.NewtonConfig(max_iters=5), ex)
    assert not rep.converged  # 5 steps do not reach ||delta||_inf <= 1e-8
    _check_records(rep, g, 5)
    uh = u.cpu().numpy()
    assert abs(np.linalg.norm(uh) - float(g["u_norm"])) <= 1e-8 * float(g["u_norm"])
    s = int(g["stride"])
    assert np.linalg.norm(uh[::s] - g["u_sample"]) <= 1e-7 * np.linalg.norm(g["u_sample"])
