"""Time pgm_matrix_upload of the cfg2 matrix from host arrays (tuning aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1906_04051_b200 as pg  # noqa: E402

ex = pg.DeviceExecutor(0)
A, b = ex.assemble_bratu(50, 6.8, device=False)
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dA = ex.upload(A)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dA.close()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"upload {1e3 * (t1 - t0):.1f} ms  destroy {1e3 * (t2 - t1):.1f} ms", flush=True)
