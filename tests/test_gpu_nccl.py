"""GPU: the NCCL transport of the multi-GPU path on one GPU.  A context with
world = 1 and an ncclUniqueId builds a 1-rank NCCL communicator through the
library's run-time binding (dlopen libnccl.so.2, ncclGetUniqueId,
ncclCommInitRank) and runs in collective mode: every reduction kernel writes
its block-reduced sums to red_out, ncclAllReduce runs on the library stream
and k_finish applies the finisher, exactly as on every rank of a multi-GPU
solve.  Results must match the reference like the single-GPU path."""
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


def test_nccl_collective_mode_cfg1(cuda, golden):
    g = golden("cfg1_defl")
    ne = 10
    uid = pg.nccl_unique_id()
    assert len(uid) == 128
    ex = pg.DeviceExecutor(0, nccl_id=uid)
    A, b = ex.assemble_bratu(ne, 6.8, device=False)
    d = pg.Deflator(pg.DeflationConfig(), ex)
    x = np.zeros(ex.n_own)
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), d, ex)
    b0 = float(g["beta0"])
    assert rep.restarts == int(g["restarts"])
    assert abs(rep.total_inner - int(g["total_inner"])) <= 1
    n = min(len(rep.monitored), len(g["monitored"]))
    assert np.max(np.abs(rep.monitored[:n] - g["monitored"][:n])) <= 1e-10 * b0
    assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])
    assert d.rank() == int(g["rank"])


def test_nccl_collective_mode_newton(cuda, golden):
    g = golden("newton_ne8")
    ex = pg.DeviceExecutor(0, nccl_id=pg.nccl_unique_id())
    u = np.zeros((2 * 8 + 1) ** 3)
    rep = pg.newton_solve(8, 6.8, u, pg.NewtonConfig(), ex)
    assert rep.converged and len(rep.iters) == len(g["inner"])
    assert np.linalg.norm(u - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])
