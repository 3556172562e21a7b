"""Golden fixtures for the full-size BASELINE configs, made by running the
REFERENCE itself (oracle/_ref, the reference sources compiled verbatim + the
Eigen shim) on this container's host cores.  Slow (tens of minutes); kept
apart from make_golden.py.

    python tests/golden/make_golden_large.py cfg3     # n_e=125, ~16M DOF
    python tests/golden/make_golden_large.py newton79 # n_e=79, 5 Newton steps

Only histories, norms and a strided sample of the solution are stored (the
full vectors are 126 MB / 32 MB); the GPU tests compare those.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import refbind as R  # noqa: E402

THREADS = os.cpu_count() or 1
SAMPLE_STRIDE = 9973


def save(name, **kw):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **kw)
    print("wrote", name, {k: (v.shape if hasattr(v, "shape") else v) for k, v in kw.items()},
          flush=True)


def cfg3():
    # BASELINE config 3: n_e=125 (15,813,251 DOF), GMRES(50) + deflation, tol 1e-10.
    # Deterministic partitioned executor: bit-identical for every thread count.
    t0 = time.time()
    A, b = R.first_newton_system(125, threads=THREADS)
    print(f"assembly {time.time() - t0:.1f} s n={A.n} nnz={A.nnz}", flush=True)
    t0 = time.time()
    r = R.solve(A, b, ne=125, threads=THREADS, m=50, rel_tol=1e-10)
    print(f"solve {time.time() - t0:.1f} s restarts={r.restarts} inner={r.total_inner}",
          flush=True)
    save("cfg3_defl", beta0=r.beta0, restarts=r.restarts, total_inner=r.total_inner,
         converged=r.converged, final_relative=r.final_relative,
         inner_restart=r.inner_restart, inner_step=r.inner_step, monitored=r.monitored,
         explicit_residual=r.explicit_residual, rank=r.rank, mu=r.mu, skipped=r.skipped,
         hist_restart=r.hist_restart, hist_r=r.hist_r, hist_mu=r.hist_mu,
         hist_theta=r.hist_theta, x_norm=np.linalg.norm(r.x), x_sample=r.x[::SAMPLE_STRIDE].copy(),
         b_norm=np.linalg.norm(b), stride=SAMPLE_STRIDE, wall_s=r.wall_s, threads=THREADS)


def newton79():
    # BASELINE config 4: 5 Newton steps on n_e=79 (4,019,679 DOF), deflated
    # GMRES(50) to 1e-10 per step (NewtonConfig defaults, newton.hpp:15-23).
    t0 = time.time()
    nw = R.newton(79, max_iters=5, threads=THREADS)
    print(f"newton {time.time() - t0:.1f} s", nw["iters"], flush=True)
    u = nw["u"]
    save("newton79", inner=np.array([i["gmres_inner"] for i in nw["iters"]]),
         restarts=np.array([i["gmres_restarts"] for i in nw["iters"]]),
         update_inf=np.array([i["update_inf"] for i in nw["iters"]]),
         residual_norm=np.array([i["residual_norm"] for i in nw["iters"]]),
         u_norm=np.linalg.norm(u), u_max=u.max(), u_sample=u[::SAMPLE_STRIDE].copy(),
         stride=SAMPLE_STRIDE, converged=nw["converged"], wall_s=nw["wall_s"],
         threads=THREADS)


if __name__ == "__main__":
    for what in sys.argv[1:] or ["cfg3", "newton79"]:
        globals()[what]()
