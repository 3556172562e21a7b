"""Break down one e2e bench step (host CSR upload + solve) (tuning aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_04051_b200 as pg  # noqa: E402

ex = pg.DeviceExecutor(0)
A, b = ex.assemble_bratu(50, 6.8, device=False)
d = pg.Deflator(pg.DeflationConfig(), ex)
cfg = pg.GmresConfig(m=50, rel_tol=1e-10)
x = np.zeros(A.n)
dA = ex.upload(A)
for i in range(3):
    d.reset()
    x[:] = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = pg.deflated_gmres(dA, b, x, cfg, d, ex)
    t1 = time.perf_counter()
    print(f"resident-matrix solve {1e3 * (t1 - t0):.1f} ms (device {rep.solve_seconds * 1e3:.1f})",
          rep.total_inner, flush=True)
for i in range(3):
    d.reset()
    x[:] = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dA2 = ex.upload(A)
    t1 = time.perf_counter()
    rep = pg.deflated_gmres(dA2, b, x, cfg, d, ex)
    t2 = time.perf_counter()
    dA2.close()
    t3 = time.perf_counter()
    print(f"upload {1e3 * (t1 - t0):.1f} solve {1e3 * (t2 - t1):.1f} (device "
          f"{rep.solve_seconds * 1e3:.1f}) close {1e3 * (t3 - t2):.1f} ms", rep.total_inner,
          flush=True)
