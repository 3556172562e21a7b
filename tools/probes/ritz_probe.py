"""Probe (PGM_TAIL_TIMING variant): k_ritz phase times per call."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1906_04051_b200 as pg  # noqa: E402
from paper_1906_04051_b200 import _capi  # noqa: E402

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ex = pg.DeviceExecutor()
A, b = ex.assemble_bratu(ne, 6.8, device=True)
dA = ex.upload(A)
x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
L = _capi.lib()
buf = (C.c_ulonglong * 16)()
d = pg.Deflator(pg.DeflationConfig(), ex)
L.pgm_debug_tail(buf)
pg.deflated_gmres(dA, b, x, pg.GmresConfig(m=50, rel_tol=1e-10), d, ex)
L.pgm_debug_tail(buf)
nc = max(1, buf[8])
print(f"n_e={ne}: {buf[8]} Ritz calls; per call: power {buf[4]/nc/1e3:.1f} us, until GJ done "
      f"{buf[5]/nc/1e3:.1f} us ({buf[13]/nc:.0f} power its), inverse iteration {buf[6]/nc/1e3:.1f} us ({buf[7]/nc:.0f} its)")
