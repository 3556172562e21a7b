"""Probe: deflation basis around the first truncation (criterion-8 protocol,
n_e=8): dump U, T, history after restarts 18..22 to gpurun_out/trunc_probe.npz."""
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
out = {}


def hook(ctx):
    r = d.rank()
    U = d.basis_matrix()
    o = np.abs(U.T @ U - np.eye(r)).max() if r else 0.0
    print(ctx.restart, ctx.steps, r, f"{o:.2e}", d.skipped_updates(), flush=True)
    if 17 <= ctx.restart <= 22:
        out[f"U{ctx.restart}"] = U.copy()
        out[f"T{ctx.restart}"] = d.T_block()


x = np.zeros(A.n)
rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=50, max_restarts=24, fixed_iterations=True),
                        d, ex, observer=hook)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/trunc_probe.npz", **out)
