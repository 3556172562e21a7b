"""The reference's own sensitivity of the Newton run (BASELINE config 4,
n_e = 79, 5 steps): per-step GMRES inner counts with the deterministic
executor (= tests/golden/newton79.npz) and the non-deterministic one
(REFD_EXEC=nondet, per-worker partial sums), all host threads.

    python tools/ref_newton_spread.py out.json
"""
import json
import os
import subprocess
import sys

code = ("import json,os,sys; sys.path.insert(0,'.'); from oracle import refbind as R; "
        "nw=R.newton(79, max_iters=5, threads=os.cpu_count()); "
        "print(json.dumps({'inner':[i['gmres_inner'] for i in nw['iters']],"
        "'wall_s':nw['wall_s']}))")
out = {}
for mode in ("det", "nondet"):
    env = dict(os.environ, REFD_EXEC=mode)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    print(mode, out[mode], flush=True)
with open(sys.argv[1] if len(sys.argv) > 1 else "ref_newton_spread.json", "w") as f:
    json.dump(out, f, indent=1)
