"""Probe: host CSR -> device SELL upload rate (pgm_matrix_upload) from pinned
and from pageable host arrays, and the value refresh (pgm_matrix_update_values)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1906_04051_b200 as pg  # noqa: E402

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 125
ex = pg.DeviceExecutor()
A, b = ex.assemble_bratu(ne, 6.8, device=False)
n, nnz = A.n, A.nnz
gb = (4 * (n + 1) + 12 * nnz) / 1e9
rp_p = torch.from_numpy(A.row_ptr.view(np.int32)).pin_memory()
ci_p = torch.from_numpy(A.col_idx.view(np.int32)).pin_memory()
va_p = torch.from_numpy(A.values).pin_memory()
Ap = pg.CsrMatrix(n, rp_p.numpy().view(np.uint32), ci_p.numpy().view(np.uint32), va_p.numpy())
for name, M in (("pinned", Ap), ("pageable", A)):
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = ex.upload(M)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        t1 = time.perf_counter()
        d.update_values(M.values)
        torch.cuda.synchronize()
        tv = time.perf_counter() - t1
        d.close()
    print(f"n_e={ne} {name}: upload {t*1e3:.1f} ms ({gb / t:.1f} GB/s), update_values "
          f"{tv*1e3:.1f} ms ({8 * nnz / 1e9 / tv:.1f} GB/s)", flush=True)
