"""Break down one e2e bench step (host CSR upload + solve) (tuning aid).

    python tools/time_e2e.py [--ne 125]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_04051_b200 as pg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ne", type=int, default=125)
a = ap.parse_args()
ex = pg.DeviceExecutor(0)
A_d, b_d = ex.assemble_bratu(a.ne, 6.8, device=True)
n, nnz = ex.n_own, A_d.nnz
rp = torch.empty(n + 1, dtype=torch.int32, pin_memory=True)
ci = torch.empty(nnz, dtype=torch.int32, pin_memory=True)
va = torch.empty(nnz, dtype=torch.float64, pin_memory=True)
rp.copy_(A_d.row_ptr)
ci.copy_(A_d.col_idx)
va.copy_(A_d.values)
b = b_d.cpu().numpy()
A = pg.CsrMatrix(n, rp.numpy().view(np.uint32), ci.numpy().view(np.uint32), va.numpy())
d = pg.Deflator(pg.DeflationConfig(), ex)
cfg = pg.GmresConfig(m=50, rel_tol=1e-10)
x = np.zeros(n)
for i in range(3):
    d.reset()
    x[:] = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dA = ex.upload(A)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rep = pg.deflated_gmres(dA, b, x, cfg, d, ex)
    t2 = time.perf_counter()
    dA.close()
    t3 = time.perf_counter()
    print(f"upload {1e3 * (t1 - t0):.1f} ms ({12 * nnz / (t1 - t0) / 1e9:.1f} GB/s of CSR) "
          f"solve {1e3 * (t2 - t1):.1f} (device {rep.solve_seconds * 1e3:.1f}) "
          f"close {1e3 * (t3 - t2):.1f} ms", rep.total_inner, flush=True)
