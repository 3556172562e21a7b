"""Probe (PGMRES_LIB = the PGM_TAIL_TIMING variant): average reduction-tail
and finisher time of the DCGS2 step SpMV at a given mesh."""
import ctypes as C
import os
import sys

import numpy as np
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
for rep in range(2):
    d = pg.Deflator(pg.DeflationConfig(), ex)
    x.zero_()
    L.pgm_debug_tail(buf)
    r = pg.deflated_gmres(dA, b, x, pg.GmresConfig(m=50, rel_tol=1e-10), d, ex)
    L.pgm_debug_tail(buf)
    nl = max(1, buf[3])
    print(f"n_e={ne} solve {r.solve_seconds*1e3:.1f} ms, {r.total_inner} steps; per step SpMV: "
          f"level1 {buf[0]/nl/1e3:.2f} us, level2 {buf[1]/nl/1e3:.2f} us, finisher "
          f"{buf[2]/nl/1e3:.2f} us over {buf[3]} launches; finisher phases (loads, serial, "
          f"coefficients, tail) " + " ".join(f"{buf[9 + q]/nl/1e3:.2f}" for q in range(4)) + " us")
