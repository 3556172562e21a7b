"""CPU, world_size 2 (gloo): the multi-GPU decomposition the CUDA path uses —
z-slab rows from pgm_partition_rows (the product's partition, = the
reference's partition_rows, parallel.cpp:50-71), local column ids shifted by
row_begin - halo_lo, 2-plane halo exchange of the SpMV input, one allreduce per
reduction family of the CGS2 step — restated in numpy over torch.distributed,
must reproduce the single-process solve.  The ncclUniqueId bootstrap (rank 0
creates, broadcast) is exercised with the same collective."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partition(n_axis, p, w):
    from paper_1906_04051_b200 import _capi

    out = _capi.Partition()
    assert _capi.lib().pgm_partition_rows(n_axis, p, w, C.byref(out)) == 0
    return out.row_begin, out.row_end, out.halo_lo, out.halo_hi


def _worker(rank, world, port, ne, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import refbind as R

        # --- bootstrap: rank 0's 128-byte id reaches every rank unchanged
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid.copy_(torch.arange(128, dtype=torch.uint8))
        dist.broadcast(uid, 0)
        assert bytes(uid.numpy()) == bytes(range(128))

        A, b = R.first_newton_system(ne)
        na = 2 * ne + 1
        rb, re, lo, hi = _partition(na, world, rank)
        n = re - rb
        shift = rb - lo
        rp = A.row_ptr[rb:re + 1].astype(np.int64) - int(A.row_ptr[rb])
        ci = A.col_idx[A.row_ptr[rb]:A.row_ptr[re]].astype(np.int64) - shift
        va = A.values[A.row_ptr[rb]:A.row_ptr[re]]
        assert ci.min() >= 0 and ci.max() < lo + n + hi  # halos cover the stencil
        import scipy.sparse as sp

        Aloc = sp.csr_matrix((va, ci, rp), shape=(n, lo + n + hi))

        def halo(own):  # [halo_lo | own | halo_hi] via point-to-point
            full = np.zeros(lo + n + hi)
            full[lo:lo + n] = own
            reqs = []
            if rank > 0:
                reqs.append(dist.isend(torch.from_numpy(own[:lo].copy()), rank - 1))
                buf_lo = torch.zeros(lo, dtype=torch.float64)
                reqs.append(dist.irecv(buf_lo, rank - 1))
            if rank < world - 1:
                reqs.append(dist.isend(torch.from_numpy(own[n - hi:].copy()), rank + 1))
                buf_hi = torch.zeros(hi, dtype=torch.float64)
                reqs.append(dist.irecv(buf_hi, rank + 1))
            for r_ in reqs:
                r_.wait()
            if rank > 0:
                full[:lo] = buf_lo.numpy()
            if rank < world - 1:
                full[lo + n:] = buf_hi.numpy()
            return full

        def allreduce(vals):
            t = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        # --- restarted GMRES with CGS2, one allreduce per reduction family
        m, tol = 20, 1e-10
        bl = b[rb:re]
        x = np.zeros(n)

        def residual():
            r = bl - Aloc @ halo(x)
            return r, np.sqrt(allreduce([r @ r])[0])

        r, beta = residual()
        beta0 = beta
        mons = []
        for restart in range(50):
            V = np.zeros((m + 1, n))
            H = np.zeros((m + 1, m))
            V[0] = r / beta
            g = np.zeros(m + 1)
            g[0] = beta
            cs, sn = np.zeros(m), np.zeros(m)
            steps = 0
            for k in range(m):
                w = Aloc @ halo(V[k])
                h1 = allreduce(V[:k + 1] @ w)
                w = w - h1 @ V[:k + 1]
                h2 = allreduce(V[:k + 1] @ w)
                w = w - h2 @ V[:k + 1]
                hn = np.sqrt(allreduce([w @ w])[0])
                H[:k + 1, k] = h1 + h2
                H[k + 1, k] = hn
                V[k + 1] = w / hn
                for i in range(k):
                    a_, b_ = H[i, k], H[i + 1, k]
                    H[i, k], H[i + 1, k] = cs[i] * a_ + sn[i] * b_, -sn[i] * a_ + cs[i] * b_
                rr = np.hypot(H[k, k], H[k + 1, k])
                cs[k], sn[k] = H[k, k] / rr, H[k + 1, k] / rr
                H[k, k], H[k + 1, k] = rr, 0.0
                g[k + 1], g[k] = -sn[k] * g[k], cs[k] * g[k]
                mons.append(abs(g[k + 1]))
                steps = k + 1
                if abs(g[k + 1]) <= tol * beta0:
                    break
            y = np.linalg.solve(np.triu(H[:steps, :steps]), g[:steps])
            x = x + y @ V[:steps]
            r, beta = residual()
            if beta <= tol * beta0:
                break
        q.put((rank, rb, x, np.array(mons), beta0))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_cgs2_gmres_matches_single_process(ref):
    from oracle import pgmres_oracle as O

    ne, world = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ne, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda t: t[0])
    x = np.concatenate([o[2] for o in outs])
    assert np.array_equal(outs[0][3], outs[1][3])  # replicated scalar recurrence
    A, b = ref.first_newton_system(ne)
    M = O.csr_matrix(A.n, A.row_ptr, A.col_idx, A.values)
    xo = np.zeros(A.n)
    rep = O.gmres_restarted(lambda v: O.spmv(M, v), None, b, xo,
                            O.GmresConfig(m=20, max_restarts=50, rel_tol=1e-10), orth="cgs2")
    assert len(outs[0][3]) == rep.total_inner
    assert np.max(np.abs(outs[0][3] - rep.monitored)) <= 1e-12 * rep.beta0
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)
