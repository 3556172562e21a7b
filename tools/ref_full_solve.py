"""Measured reference time-to-solution at BASELINE config 3 on the GPU box's
host: the reference's deflated_gmres (oracle/_ref, its own sources) run to
rel_tol 1e-10 on the n_e = 125 first Newton system with all host threads,
plus a p = 1 sample (one fixed restart cycle, one thread).  Writes one JSON
object (profiles/r2_reference_cfg3_full.json).

    python tools/ref_full_solve.py gpurun_out/ref_full_cfg3.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refbind as R  # noqa: E402

ne, m, tol = 125, 50, 1e-10
th = min(os.cpu_count() or 1, 2 * ne + 1)
t0 = time.time()
A, b = R.first_newton_system(ne, threads=th)
t_asm = time.time() - t0
r = R.solve(A, b, ne=ne, threads=th, m=m, rel_tol=tol)
out = {"what": "reference deflated GMRES(50) full tolerance solve, n_e=125 (BASELINE config 3)",
       "threads": th, "assembly_s": round(t_asm, 2), "solve_s": round(r.wall_s, 2),
       "restarts": r.restarts, "total_inner": int(r.total_inner),
       "final_relative": r.final_relative, "iter_per_s": round(r.total_inner / r.wall_s, 4),
       "cpu_model": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")}
print(json.dumps(out), flush=True)
del A
S1 = R.RefSession(ne, threads=1, assembly_threads=th)
r1 = S1.run(m=m, max_restarts=1, fixed_iterations=True)
out["p1"] = {"threads": 1, "sample": "1 fixed restart cycle from x0 = 0 (rank 0)",
             "inner": int(r1.total_inner), "wall_s": round(r1.wall_s, 2),
             "iter_per_s": round(r1.total_inner / r1.wall_s, 4)}
out["p1"]["all_threads_vs_p1"] = round(out["iter_per_s"] / out["p1"]["iter_per_s"], 2)
with open(sys.argv[1] if len(sys.argv) > 1 else "ref_full_cfg3.json", "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out), flush=True)
