"""Round-2 parity fixtures: solution vectors checked at the north star's 1e-8
with no slack.  Made by running the REFERENCE (oracle/_ref: its sources
compiled verbatim + the Eigen shim) on this container's host cores.

    python tests/golden/make_golden_r2.py cfg2 sweep31 cfg3

* cfg2_full.npz  — n_e=50 (1,030,301 DOF), GMRES(50) deflated AND undeflated:
  histories plus the FULL solution vectors.
* sweep_ne31.npz — BASELINE config 5's smallest mesh (n_e=31, 250,047 DOF),
  m in {20, 50, 100} x deflation on/off: histories, x every 4th entry and the
  l2 norm of x on every node plane.
* cfg3_x.npz     — n_e=125 (15.8 M DOF), deflated GMRES(50): histories, x
  every 16th entry and per-plane l2 norms (the full vector is 126 MB).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import refbind as R  # noqa: E402

THREADS = os.cpu_count() or 1


def plane_norms(x, ne):
    na = 2 * ne + 1
    return np.linalg.norm(x.reshape(na, na * na), axis=1)


def hist(prefix, r):
    return {prefix + "beta0": r.beta0, prefix + "restarts": r.restarts,
            prefix + "total_inner": r.total_inner, prefix + "converged": r.converged,
            prefix + "breakdown": r.breakdown, prefix + "final_relative": r.final_relative,
            prefix + "monitored": r.monitored, prefix + "explicit": r.explicit_residual,
            prefix + "rank": r.rank, prefix + "mu": r.mu, prefix + "hist_r": r.hist_r,
            prefix + "x_norm": np.linalg.norm(r.x)}


def save(name, out):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print("wrote", name, flush=True)


def cfg2():
    A, b = R.first_newton_system(50, threads=THREADS)
    out = {}
    for defl in (True, False):
        t0 = time.time()
        r = R.solve(A, b, ne=50, threads=THREADS, m=50, rel_tol=1e-10, deflation=defl)
        key = "defl_" if defl else "plain_"
        print(key, r.restarts, r.total_inner, f"{time.time() - t0:.1f} s", flush=True)
        out.update(hist(key, r))
        out[key + "x"] = r.x
    save("cfg2_full", out)


def sweep31():
    ne = 31
    A, b = R.first_newton_system(ne, threads=THREADS)
    out = {}
    for m in (20, 50, 100):
        for defl in (True, False):
            r = R.solve(A, b, m=m, rel_tol=1e-10, max_restarts=300, deflation=defl, ne=ne,
                        threads=THREADS)
            key = f"m{m}_{'defl' if defl else 'plain'}_"
            out.update(hist(key, r))
            out[key + "x_stride4"] = r.x[::4].copy()
            out[key + "x_planes"] = plane_norms(r.x, ne)
            print(key, r.restarts, r.total_inner, r.rank, flush=True)
    save("sweep_ne31", out)


def cfg3():
    t0 = time.time()
    A, b = R.first_newton_system(125, threads=THREADS)
    print(f"assembly {time.time() - t0:.1f} s", flush=True)
    t0 = time.time()
    r = R.solve(A, b, ne=125, threads=THREADS, m=50, rel_tol=1e-10)
    print(f"solve {time.time() - t0:.1f} s restarts={r.restarts} inner={r.total_inner}",
          flush=True)
    out = hist("", r)
    out["x_stride16"] = r.x[::16].copy()
    out["x_planes"] = plane_norms(r.x, 125)
    out["wall_s"] = r.wall_s
    out["threads"] = THREADS
    save("cfg3_x", out)


if __name__ == "__main__":
    for what in sys.argv[1:] or ["cfg2", "sweep31", "cfg3"]:
        globals()[what]()
