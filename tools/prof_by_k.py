"""Per-launch CUDA-event profile of one cfg2 deflated solve, grouped by kernel
class and Arnoldi step k (tuning aid; numbers are not bench values).

    python tools/prof_by_k.py [--ne 50] [--m 50]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_04051_b200 as pg  # noqa: E402

NAMES = ["step_spmv", "cgs2_B", "cgs2_C", "x_update", "ritz", "push", "push_spmv", "rotate",
         "residual", "other"]
ap = argparse.ArgumentParser()
ap.add_argument("--ne", type=int, default=50)
ap.add_argument("--m", type=int, default=50)
ap.add_argument("--fixed", type=int, default=0, help="fixed-iteration mode with this many restarts")
a = ap.parse_args()
ex = pg.DeviceExecutor(0)
A, b = ex.assemble_bratu(a.ne, 6.8, device=True)
dA = ex.upload(A)
x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
d = pg.Deflator(pg.DeflationConfig(), ex)
for prof in (False, True):
    d.reset()
    x.zero_()
    ex.set_profiling(prof)
    torch.cuda.synchronize()
    cfg = (pg.GmresConfig(m=a.m, max_restarts=a.fixed, fixed_iterations=True) if a.fixed
           else pg.GmresConfig(m=a.m, rel_tol=1e-10))
    rep = pg.deflated_gmres(dA, b, x, cfg, d, ex)
print("solve", rep.solve_seconds * 1e3, "ms", rep.restarts, rep.total_inner)
cls, cyc, kk, ms = ex.profile()
n = ex.n_own
agg = collections.defaultdict(list)
for c, y, k, t in zip(cls, cyc, kk, ms):
    if int(y) >= rep.restarts - 1:
        continue
    agg[(int(c), int(k))].append(t)
for c in (0, 1, 2):
    print(NAMES[c])
    for k in range(a.m):
        if (c, k) in agg:
            t = np.median(agg[(c, k)])
            j = k + 1
            byts = {1: 8 * n * (j + 2), 2: 8 * n * (j + 2 + 5)}.get(c, 0)
            gb = f"{byts / (t * 1e-3) / 1e9:7.0f} GB/s" if byts else ""
            print(f"  k={k:3d} {t * 1e3:8.1f} us {gb}")
tot = collections.defaultdict(float)
for c, t in zip(cls, ms):
    tot[NAMES[int(c)]] += t
print({k: round(v, 3) for k, v in tot.items()}, "sum", round(sum(tot.values()), 3))
