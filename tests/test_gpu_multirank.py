"""GPU: the multi-rank path (z-slab rows, halo planes, per-reduction allreduce
+ replicated finisher) run as W ranks on ONE GPU through the in-process
loopback communicator (one host thread per rank).  Kernels, partition
(partition_rows, parallel.cpp:50-71) and collective placement are the
production world > 1 code; the allreduce runs either fused inside the
reduction kernels over peer memory (the in-kernel protocol used with CUDA IPC
windows across GPUs) or host-staged in place of NCCL."""
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


@pytest.fixture(params=["peer", "host"])
def transport(request, monkeypatch):
    """peer: the fused in-kernel allreduce over peer memory (default for
    in-process ranks); host: the host-staged loopback collective (the NCCL
    code path's allreduce_red + k_finish placement)."""
    monkeypatch.setenv("PGMRES_PEER", "1" if request.param == "peer" else "0")
    return request.param


def run_ranks(world, fn):
    grp = pg.LoopbackGroup(world)
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


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_spmv_bitexact(cuda, ref, world):
    ne = 10
    na = 2 * ne + 1
    Ar, _ = ref.first_newton_system(ne)
    x = np.random.default_rng(world).uniform(-1, 1, Ar.n)

    def rank(r, grp):
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
        A, _ = ex.assemble_bratu(ne, 6.8, device=False)
        p = ex.partition()
        dA = ex.upload(A)
        y = ex.spmv(dA, x[p["row_begin"]:p["row_end"]].copy())
        return p, y

    res = run_ranks(world, rank)
    y = np.concatenate([yy for _, yy in res])
    assert np.array_equal(y, ref.spmv(Ar, x))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_multirank_deflated_cfg1(cuda, golden, world, transport):
    ne = 10
    na = 2 * ne + 1
    g = golden("cfg1_defl")

    def rank(r, grp):
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
        A, b = ex.assemble_bratu(ne, 6.8, device=False)
        d = pg.Deflator(pg.DeflationConfig(), ex)
        x = np.zeros(ex.n_own)
        rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), d, ex)
        return rep, x, d.rank(), d.mu()

    res = run_ranks(world, rank)
    x = np.concatenate([rr[1] for rr in res])
    rep0 = res[0][0]
    for rep, _, rk, mu in res:  # replicated scalar state
        assert rep.total_inner == rep0.total_inner and rk == res[0][2] and mu == res[0][3]
        assert np.array_equal(rep.monitored, rep0.monitored)
    b0 = float(g["beta0"])
    assert rep0.restarts == int(g["restarts"])
    assert abs(rep0.total_inner - int(g["total_inner"])) <= 1
    n = min(len(rep0.monitored), len(g["monitored"]))
    assert np.max(np.abs(rep0.monitored[:n] - g["monitored"][:n])) <= 1e-10 * b0
    assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])
    assert res[0][2] == int(g["rank"])


def test_multirank_truncation_run(cuda, golden, transport):
    ne, world = 10, 2
    na = 2 * ne + 1
    g = golden("ne10_m4_trunc")

    def rank(r, grp):
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
        A, b = ex.assemble_bratu(ne, 6.8, device=False)
        d = pg.Deflator(pg.DeflationConfig(), ex)
        x = np.zeros(ex.n_own)
        rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=4, max_restarts=24,
                                                        fixed_iterations=True), d, ex)
        return rep, x, [h.r for h in d.history()], d.T_block()

    res = run_ranks(world, rank)
    x = np.concatenate([rr[1] for rr in res])
    assert res[0][2] == list(g["hist_r"])
    assert np.abs(res[0][3] - g["T"]).max() <= 1e-8 * np.abs(g["T"]).max()
    assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])


def test_multirank_newton_ne8(cuda, golden, transport):
    """The device-resident Newton driver on 2 z-slab ranks: every rank
    assembles its rows from the global iterate, solves its share and keeps
    its halo planes of u current; result identical to the reference's."""
    ne, world = 8, 2
    na = 2 * ne + 1
    g = golden("newton_ne8")

    def rank(r, grp):
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
        u = np.zeros(na ** 3)
        rep = pg.newton_solve(ne, 6.8, u, pg.NewtonConfig(), ex)
        p = ex.partition()
        return rep, u[p["row_begin"]:p["row_end"]].copy()

    res = run_ranks(world, rank)
    u = np.concatenate([rr[1] for rr in res])
    rep = res[0][0]
    assert rep.converged and len(rep.iters) == len(g["inner"])
    assert [it.gmres_inner for it in rep.iters] == [it.gmres_inner for it in res[1][0].iters]
    assert np.all(np.abs(np.array([it.gmres_inner for it in rep.iters]) - g["inner"]) <= 3)
    assert np.linalg.norm(u - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])


@pytest.mark.slow
@pytest.mark.parametrize("world", [4])
def test_multirank_cfg2_size(cuda, golden, world, transport):
    """BASELINE config 2 (n_e = 50, 1.03 M DOF) on W = 4 z-slab ranks (one GPU,
    loopback): the per-rank size of config 3 split over 8 GPUs is in this
    regime.  Same iteration count, histories within 1e-10 * beta0, the full
    solution within 1e-8 of the reference's."""
    ne = 50
    na = 2 * ne + 1
    g = golden("cfg2_full")

    def rank(r, grp):
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
        A, b = ex.assemble_bratu(ne, 6.8, device=True)
        d = pg.Deflator(pg.DeflationConfig(), ex)
        x = cuda.zeros(ex.n_own, dtype=cuda.float64, device="cuda")
        rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=50, rel_tol=1e-10), d, ex)
        return rep, x.cpu().numpy(), d.rank()

    res = run_ranks(world, rank)
    x = np.concatenate([rr[1] for rr in res])
    rep0 = res[0][0]
    for rep, _, rk in res:
        assert rep.total_inner == rep0.total_inner and rk == res[0][2]
    b0 = float(g["defl_beta0"])
    assert abs(rep0.total_inner - int(g["defl_total_inner"])) <= 1
    n = min(len(rep0.monitored), len(g["defl_monitored"]))
    assert np.max(np.abs(rep0.monitored[:n] - g["defl_monitored"][:n])) <= 1e-10 * b0
    assert np.linalg.norm(x - g["defl_x"]) <= 1e-8 * np.linalg.norm(g["defl_x"])
    assert res[0][2] == int(g["defl_rank"])


@pytest.mark.parametrize("defl", [True, False])
def test_multirank_m100(cuda, golden, transport, defl):
    """BASELINE's largest restart length (m = 100, n_e = 25 sweep golden) on
    W = 2 ranks.  On the peer transport 2m + 2 + r_max + 1 exceeds the window
    slot, so the solve runs the CGS2 step (two reductions per step) there."""
    ne, world = 25, 2
    na = 2 * ne + 1
    g = golden("sweep_ne25")
    key = f"m100_{'defl' if defl else 'plain'}"

    def rank(r, grp):
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
        A, b = ex.assemble_bratu(ne, 6.8, device=True)
        x = cuda.zeros(ex.n_own, dtype=cuda.float64, device="cuda")
        cfg = pg.GmresConfig(m=100, max_restarts=200, rel_tol=1e-10)
        if defl:
            rep = pg.deflated_gmres(A, b, x, cfg, pg.Deflator(pg.DeflationConfig(), ex), ex)
        else:
            rep = pg.gmres_restarted(A, None, b, x, cfg, ex)
        return rep, x.cpu().numpy()

    res = run_ranks(world, rank)
    x = np.concatenate([rr[1] for rr in res])
    rep0 = res[0][0]
    b0 = float(g[key + "_beta0"])
    assert abs(rep0.total_inner - int(g[key + "_total_inner"])) <= 1
    n = min(len(rep0.monitored), len(g[key + "_monitored"]))
    assert np.max(np.abs(rep0.monitored[:n] - g[key + "_monitored"][:n])) <= 1e-10 * b0
    assert abs(np.linalg.norm(x) - float(g[key + "_x_norm"])) <= 1e-8 * float(g[key + "_x_norm"])
    assert np.linalg.norm(x[::97] - g[key + "_x_sample"]) <= 1e-8 * np.linalg.norm(
        g[key + "_x_sample"])
