"""Probe: loopback W=2 SpMV through the peer-memory halo mailboxes."""
import os
import sys
import threading

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1906_04051_b200 as pg  # noqa: E402
from oracle import refbind as R  # noqa: E402

ne, world = int(sys.argv[1]) if len(sys.argv) > 1 else 4, 2
na = 2 * ne + 1
Ar, _ = R.first_newton_system(ne)
x = np.random.default_rng(1).uniform(-1, 1, Ar.n)
yref = R.spmv(Ar, x)
grp = pg.LoopbackGroup(world)
out = {}


def rank(r):
    ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
    A, _ = ex.assemble_bratu(ne, 6.8, device=False)
    p = ex.partition()
    dA = ex.upload(A)
    for rep in range(3):
        y = ex.spmv(dA, x[p["row_begin"]:p["row_end"]].copy())
        out[(r, rep)] = (p, y)


th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
for t in th:
    t.start()
for t in th:
    t.join()
for rep in range(3):
    for r in range(world):
        p, y = out[(r, rep)]
        d = np.abs(y - yref[p["row_begin"]:p["row_end"]])
        bad = np.nonzero(d > 0)[0]
        print(rep, r, p, "bad rows", len(bad), bad[:5], bad[-5:] if len(bad) else "")
