"""Golden fixtures for BASELINE config 5's restart-length sweep (m in {20, 50,
100}, deflation on/off) on n_e = 25 (132,651 DOF), made by running the
REFERENCE (oracle/_ref: its sources compiled verbatim + the Eigen shim).

    python tests/golden/make_golden_sweep.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import refbind as R  # noqa: E402

THREADS = min(8, os.cpu_count() or 1)


def main():
    A, b = R.first_newton_system(25, threads=THREADS)
    out = {}
    for m in (20, 100):
        for defl in (True, False):
            r = R.solve(A, b, m=m, rel_tol=1e-10, max_restarts=200, deflation=defl, ne=25,
                        threads=THREADS)
            key = f"m{m}_{'defl' if defl else 'plain'}"
            out[key + "_beta0"] = r.beta0
            out[key + "_restarts"] = r.restarts
            out[key + "_total_inner"] = r.total_inner
            out[key + "_monitored"] = r.monitored
            out[key + "_explicit"] = r.explicit_residual
            out[key + "_x_norm"] = np.linalg.norm(r.x)
            out[key + "_x_sample"] = r.x[::97].copy()
            print(key, r.restarts, r.total_inner, r.rank, flush=True)
    np.savez_compressed(os.path.join(HERE, "sweep_ne25.npz"), **out)


if __name__ == "__main__":
    main()
