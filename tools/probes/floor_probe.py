"""Probe: deflated GMRES(50), 100 fixed restarts at n_e=8 (criterion 2/8
protocol) on the device — restarts, breakdown, last cycles' step counts and
monitored residuals, for the DCGS2 and CGS2 steps."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1906_04051_b200 as pg  # noqa: E402
from oracle import refbind as R  # noqa: E402

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 8
Ar, b = R.first_newton_system(ne)
A = pg.CsrMatrix(Ar.n, Ar.row_ptr, Ar.col_idx, Ar.values)
ex = pg.DeviceExecutor()
x = np.zeros(A.n)
d = pg.Deflator(pg.DeflationConfig(r_max=20))
rep = pg.deflated_gmres(A, b, x, pg.GmresConfig(m=50, max_restarts=100, fixed_iterations=True), d, ex)
steps = np.bincount(rep.inner_restart)
print("restarts", rep.restarts, "inner", rep.total_inner, "breakdown", rep.breakdown,
      "final", rep.final_relative, "rank", d.rank())
print("steps of last cycles", steps[-8:])
print("explicit tail", rep.explicit_residual[-8:] / rep.beta0)
last = rep.inner_restart == rep.restarts - 1
print("monitored last cycle", rep.monitored[last][-6:] / rep.beta0)
