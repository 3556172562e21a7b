import os, sys, threading
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1906_04051_b200 as pg
world, ne = 2, 10
na = 2 * ne + 1
grp = pg.LoopbackGroup(world)
res = {}
def body(r):
    try:
        ex = pg.DeviceExecutor(0, n_global=na ** 3, n_axis=na, rank=r, world=world, loopback=grp)
        A, b = ex.assemble_bratu(ne, 6.8, device=False)
        d = pg.Deflator(pg.DeflationConfig(), ex)
        x = np.zeros(ex.n_own)
        rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), d, ex)
        res[r] = (rep.total_inner, rep.restarts)
    except Exception as e:
        res[r] = repr(e)
th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
[t.start() for t in th]; [t.join(timeout=120) for t in th]
print(res)
