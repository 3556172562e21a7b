"""Parity + speed check of the DCGS2 device path (PGMRES_DCGS2=1) against the
reference goldens (tuning aid)."""
import os
import sys
import time

os.environ.setdefault("PGMRES_DCGS2", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_04051_b200 as pg  # noqa: E402


def load(n):
    z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", n + ".npz"))
    return {k: z[k] for k in z.files}


for ne, m, key, defl in [(10, 30, "cfg1_defl", True), (10, 30, "cfg1_plain", False),
                         (50, 50, "cfg2_defl", True)]:
    g = load(key)
    ex = pg.DeviceExecutor(0)
    A, b = ex.assemble_bratu(ne, 6.8, device=True)
    x = torch.zeros(ex.n_own, dtype=torch.float64, device="cuda")
    cfg = pg.GmresConfig(m=m, rel_tol=1e-10)
    d = pg.Deflator(pg.DeflationConfig(), ex)
    for rep_i in range(2):
        x.zero_()
        d.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = pg.deflated_gmres(A, b, x, cfg, d, ex) if defl else pg.gmres_restarted(A, None, b, x, cfg, ex)
        t = time.perf_counter() - t0
    mon = rep.monitored
    gm = g["monitored"]
    n = min(len(mon), len(gm))
    b0 = float(g["beta0"])
    xn = float(np.linalg.norm(x.cpu().numpy()))
    gx = float(g["x_norm"]) if "x_norm" in g else float(np.linalg.norm(g["x"]))
    print(key, "restarts", rep.restarts, int(g["restarts"]), "inner", rep.total_inner,
          int(g["total_inner"]), "maxdiff/b0 %.2e" % (np.max(np.abs(mon[:n] - gm[:n])) / b0),
          "xnorm rel %.2e" % (abs(xn - gx) / gx), "time %.1f ms" % (1e3 * t),
          "it/s %.0f" % (rep.total_inner / t), flush=True)
