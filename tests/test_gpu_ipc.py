"""GPU: the cross-process peer transport — two PROCESSES (one rank each) on
one GPU, no NCCL (peer_only): halo planes and every reduction go through
the other process's CUDA-IPC-mapped window (pgm_peer_export /
pgm_peer_import, k_halo_push / k_halo_pull, the in-kernel peer allreduce).
Without MPS the two contexts are time-sliced, so every cross-rank wait is
resolved at a context switch: slow, but it exercises exactly the code path
one process per GPU uses over NVLink.  Result: the reference's cfg1 solve."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, ne, q_handles, q_all, q_res):
    os.environ["CUDA_MODULE_LOADING"] = "EAGER"
    sys.path.insert(0, ROOT)
    try:
        import paper_1906_04051_b200 as pg

        na = 2 * ne + 1
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=rank, world=world,
                               peer_only=True)
        q_handles.put((rank, ex.peer_export()))
        ex.peer_import(q_all.get(timeout=120))
        A, b = ex.assemble_bratu(ne, 6.8, device=False)
        x = np.zeros(ex.n_own)
        d = pg.Deflator(pg.DeflationConfig(), ex)
        rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), d, ex)
        q_res.put((rank, None, rep.total_inner, rep.monitored, x, rep.beta0, d.rank()))
    except Exception as e:  # noqa: BLE001
        q_res.put((rank, repr(e), None, None, None, None, None))


def test_two_processes_one_gpu_peer_transport(golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    world, ne = 2, 10
    q_handles, q_res = ctx.Queue(), ctx.Queue()
    q_all = [ctx.Queue() for _ in range(world)]
    procs = [ctx.Process(target=_worker, args=(r, world, ne, q_handles, q_all[r], q_res))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        hs = dict(q_handles.get(timeout=300) for _ in range(world))
        for r in range(world):
            q_all[r].put([hs[q] for q in range(world)])
        res = dict((r[0], r) for r in (q_res.get(timeout=600) for _ in range(world)))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert res[r][1] is None, res[r][1]
    g = golden("cfg1_defl")
    b0 = float(g["beta0"])
    rep0, rep1 = res[0], res[1]
    assert rep0[2] == rep1[2] and rep0[6] == rep1[6]
    assert np.array_equal(rep0[3], rep1[3])  # replicated scalar state
    assert abs(rep0[2] - int(g["total_inner"])) <= 1
    n = min(len(rep0[3]), len(g["monitored"]))
    assert np.max(np.abs(rep0[3][:n] - g["monitored"][:n])) <= 1e-10 * b0
    x = np.concatenate([rep0[4], rep1[4]])
    assert np.linalg.norm(x - g["x"]) <= 1e-8 * np.linalg.norm(g["x"])
