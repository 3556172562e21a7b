"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself
(oracle/_ref: /root/reference/proj/src compiled verbatim + the Eigen shim).

    python tests/golden/make_golden.py

Every fixture records the reference's outputs on a deterministic input (the
first Newton system J(0) x = -R(0) at lambda = 6.8, x0 = 0, unless noted).
The reference run uses the deterministic partitioned executor
(Executor(partition_rows(mesh, p), true)), whose reductions are bit-identical
for every worker count (test_parallel.cpp:137-157)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import refbind as R  # noqa: E402

THREADS = min(8, os.cpu_count() or 1)


def save(name, **kw):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **kw)
    print("wrote", name, {k: (v.shape if hasattr(v, "shape") else v) for k, v in kw.items()})


def solve_record(A, b, ne, **kw):
    r = R.solve(A, b, ne=ne, threads=min(THREADS, 2 * ne + 1), **kw)
    return dict(beta0=r.beta0, restarts=r.restarts, total_inner=r.total_inner,
                converged=r.converged, breakdown=r.breakdown, final_relative=r.final_relative,
                inner_restart=r.inner_restart, inner_step=r.inner_step, monitored=r.monitored,
                explicit_residual=r.explicit_residual, rank=r.rank, mu=r.mu, skipped=r.skipped,
                hist_restart=r.hist_restart, hist_r=r.hist_r, hist_mu=r.hist_mu,
                hist_theta=r.hist_theta, x=r.x,
                T=r.T if r.T is not None else np.zeros((0, 0)))


def main():
    # cfg1: n_e=10, GMRES(30) + deflation, tol 1e-10 (BASELINE config 1)
    A, b = R.first_newton_system(10)
    save("cfg1_defl", **solve_record(A, b, 10, m=30, rel_tol=1e-10))
    save("cfg1_plain", **solve_record(A, b, 10, m=30, rel_tol=1e-10, deflation=False))
    # fixed-iteration deflated run long enough to truncate (r reaches 21)
    A4, b4 = R.first_newton_system(4)
    save("ne4_fixed_trunc", **solve_record(A4, b4, 4, m=10, max_restarts=26,
                                           fixed_iterations=True))
    # truncation well above the rounding floor: T comparable after 4 truncations
    save("ne10_m4_trunc", **solve_record(A, b, 10, m=4, max_restarts=24, fixed_iterations=True))
    # n_e=2 (45 free DOF): dense-LU equivalence and Krylov exhaustion
    A2, b2 = R.first_newton_system(2)
    save("ne2_system", row_ptr=A2.row_ptr, col_idx=A2.col_idx, values=A2.values, rhs=b2)
    save("ne2_defl", **solve_record(A2, b2, 2, m=50, rel_tol=1e-12))
    # criterion 10: spectral action on diag(1..50), GMRES(8) x 5 fixed
    D = R.diag_csr(np.arange(1, 51))
    r = R.solve(D, np.full(50, 1 / np.sqrt(50)), m=8, max_restarts=5, fixed_iterations=True)
    save("crit10_diag", rank=r.rank, mu=r.mu, hist_r=r.hist_r, hist_mu=r.hist_mu,
         hist_theta=r.hist_theta, x=r.x, monitored=r.monitored,
         explicit_residual=r.explicit_residual, T=r.T)
    # criterion 3 mid-flight: n_e=25, GMRES(50), 3 fixed restarts
    A25, b25 = R.first_newton_system(25, threads=THREADS)
    d = R.solve(A25, b25, m=50, max_restarts=3, fixed_iterations=True, ne=25, threads=THREADS)
    p = R.solve(A25, b25, m=50, max_restarts=3, fixed_iterations=True, deflation=False, ne=25,
                threads=THREADS)
    save("crit3_ne25", defl_explicit=d.explicit_residual, plain_explicit=p.explicit_residual,
         defl_monitored=d.monitored, plain_monitored=p.monitored, beta0=d.beta0)
    # Newton n_e=8 (criterion 7)
    nw = R.newton(8)
    save("newton_ne8", inner=np.array([i["gmres_inner"] for i in nw["iters"]]),
         restarts=np.array([i["gmres_restarts"] for i in nw["iters"]]),
         update_inf=np.array([i["update_inf"] for i in nw["iters"]]),
         residual_norm=np.array([i["residual_norm"] for i in nw["iters"]]),
         u=nw["u"], converged=nw["converged"])
    # cfg2 summary (n_e=50, GMRES(50) + deflation, tol 1e-10, BASELINE config 2)
    A50, b50 = R.first_newton_system(50, threads=THREADS)
    rec = solve_record(A50, b50, 50, m=50, rel_tol=1e-10)
    x = rec.pop("x")
    rec["x_norm"] = np.linalg.norm(x)
    rec["x_sample"] = x[::997].copy()
    rec["b_norm"] = np.linalg.norm(b50)
    rec["nnz"] = A50.nnz
    save("cfg2_defl", **rec)


if __name__ == "__main__":
    main()
