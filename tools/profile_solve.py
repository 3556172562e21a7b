"""Run cfg2 deflated solves for ncu captures (no timing is reported from here).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_solve.py
    ncu --set full --clock-control none --import-source on -k regex:StepEpi \
        -s 60 -c 1 -o gpurun_out/step_spmv python tools/profile_solve.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1906_04051_b200 as pg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ne", type=int, default=50)
ap.add_argument("--m", type=int, default=50)
ap.add_argument("--solves", type=int, default=1)
a = ap.parse_args()
ex = pg.DeviceExecutor(0)
A, b = ex.assemble_bratu(a.ne, 6.8, device=True)
dA = ex.upload(A)
x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
d = pg.Deflator(pg.DeflationConfig(), ex)
for _ in range(a.solves):
    d.reset()
    x.zero_()
    torch.cuda.synchronize()
    rep = pg.deflated_gmres(dA, b, x, pg.GmresConfig(m=a.m, rel_tol=1e-10), d, ex)
    print("restarts", rep.restarts, "inner", rep.total_inner, "launches", ex.launch_count())
