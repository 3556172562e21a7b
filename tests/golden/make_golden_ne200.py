"""Golden fixture for BASELINE config 5's largest mesh, n_e = 200 ("8000^2":
64,481,201 DOF, 4,073,625,625 nnz — 32-bit column ids on the device), made
by running the REFERENCE (oracle/_ref: its sources compiled verbatim + the
Eigen shim).  The CSR alone is 49 GB, so this runs on the GPU box's host
(196 GB RAM, 16 cores), not in the build container:

    gpurun -- python tests/golden/make_golden_ne200.py gpurun_out/ne200.npz

Workload: deflated GMRES(20), 2 fixed restart cycles (fixed_iterations), x0 = 0,
deterministic partitioned executor on all host threads.  Stored: the
histories, the deflation history, x every 64th entry, per-plane l2 norms of x,
and the reference's wall time.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import refbind as R  # noqa: E402

NE, M, CYCLES = 200, 20, 2


def main(out):
    threads = os.cpu_count() or 1
    t0 = time.time()
    A, b = R.first_newton_system(NE, threads=threads)
    t_asm = time.time() - t0
    print(f"assembly {t_asm:.1f} s n={A.n} nnz={A.nnz}", flush=True)
    t0 = time.time()
    r = R.solve(A, b, ne=NE, threads=threads, m=M, max_restarts=CYCLES, fixed_iterations=True,
                deflation=True)
    t_solve = time.time() - t0
    print(f"solve {t_solve:.1f} s restarts={r.restarts} inner={r.total_inner} rank={r.rank}",
          flush=True)
    na = 2 * NE + 1
    np.savez_compressed(
        out, ne=NE, m=M, cycles=CYCLES, n=A.n, nnz=A.nnz, beta0=r.beta0, restarts=r.restarts,
        total_inner=r.total_inner, monitored=r.monitored, explicit=r.explicit_residual,
        rank=r.rank, mu=r.mu, hist_r=r.hist_r, hist_mu=r.hist_mu, hist_theta=r.hist_theta,
        x_norm=np.linalg.norm(r.x), x_stride64=r.x[::64].copy(),
        x_planes=np.linalg.norm(r.x.reshape(na, na * na), axis=1), b_norm=np.linalg.norm(b),
        assembly_s=t_asm, solve_s=t_solve, wall_s=r.wall_s, threads=threads)
    print("wrote", out, flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "ne200_fixed.npz"))
