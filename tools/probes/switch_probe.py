"""Probe: DCGS2 -> CGS2 switch mid-solve (PGMRES_DC_SWITCH_AT) against the
reference at cfg1 (n_e=10, GMRES(30) deflated) and plain."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1906_04051_b200 as pg  # noqa: E402
from oracle import refbind as R  # noqa: E402

Ar, b = R.first_newton_system(10)
A = pg.CsrMatrix(Ar.n, Ar.row_ptr, Ar.col_idx, Ar.values)
for defl in (True, False):
    r = R.solve(Ar, b, m=30, rel_tol=1e-10, deflation=defl)
    ex = pg.DeviceExecutor()
    x = np.zeros(A.n)
    cfg = pg.GmresConfig(m=30, rel_tol=1e-10)
    rep = (pg.deflated_gmres(A, b, x, cfg, pg.Deflator(), ex) if defl
           else pg.gmres_restarted(A, None, b, x, cfg, ex))
    n = min(len(rep.monitored), len(r.monitored))
    print(os.environ.get("PGMRES_DC_SWITCH_AT"), defl, rep.restarts, rep.total_inner, r.restarts,
          r.total_inner, "dmon", np.abs(rep.monitored[:n] - r.monitored[:n]).max() / r.beta0,
          "dx", np.linalg.norm(x - r.x) / np.linalg.norm(r.x))
