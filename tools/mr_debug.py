import sys, threading, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1906_04051_b200 as pg
ne, world = 10, 2
na = 2*ne+1
grp = pg.LoopbackGroup(world)
res = {}
def rank(r):
    ex = pg.DeviceExecutor(0, n_global=na**3, n_axis=na, rank=r, world=world, loopback=grp)
    A, b = ex.assemble_bratu(ne, 6.8, device=False)
    print("rank", r, "assembled", A.n, flush=True)
    x = np.zeros(ex.n_own)
    rep = pg.gmres_restarted(A, None, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), ex)
    print("rank", r, "plain", rep.restarts, rep.total_inner, flush=True)
    d = pg.Deflator(pg.DeflationConfig(), ex)
    x = np.zeros(ex.n_own)
    rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=30, rel_tol=1e-10), d, ex)
    print("rank", r, "defl", rep.restarts, rep.total_inner, flush=True)
th=[threading.Thread(target=rank,args=(r,)) for r in range(world)]
[t.start() for t in th]; [t.join() for t in th]
