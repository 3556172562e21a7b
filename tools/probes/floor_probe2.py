"""Probe: per-cycle audit (steps, explicit residual, rank, ||U^T U - I||) of the
criterion-8 protocol at n_e=8 on the device."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1906_04051_b200 as pg  # noqa: E402
from oracle import refbind as R  # noqa: E402

Ar, b = R.first_newton_system(8)
A = pg.CsrMatrix(Ar.n, Ar.row_ptr, Ar.col_idx, Ar.values)
ex = pg.DeviceExecutor()
d = pg.Deflator(pg.DeflationConfig(r_max=20))
rows = []


def hook(ctx):
    r = d.rank()
    U = d.basis_matrix()
    o = np.abs(U.T @ U - np.eye(r)).max() if r else 0.0
    rows.append((ctx.restart, ctx.steps, r, o))


x = np.zeros(A.n)
rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=50, max_restarts=100, fixed_iterations=True),
                        d, ex, observer=hook)
ex_res = rep.explicit_residual / rep.beta0
for (rs, st, r, o) in rows:
    if rs >= 85 or o > 1e-10 or st != 50:
        print(rs, st, r, f"{o:.2e}", f"{ex_res[rs]:.3e}")
