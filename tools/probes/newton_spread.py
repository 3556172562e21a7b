"""Probe: per-step GMRES inner counts of the device Newton run at BASELINE
config 4 (n_e = 79, 5 steps) for the DCGS2 and the CGS2 step: the device's
own sensitivity of the late, near-stagnating solves to rounding."""
import json
import os
import subprocess
import sys

code = ("import sys,json,numpy as np; sys.path.insert(0,'.'); import paper_1906_04051_b200 as pg; "
        "ex=pg.DeviceExecutor(); import torch; "
        "u=torch.zeros(159**3,dtype=torch.float64,device='cuda'); "
        "r=pg.newton_solve(79,6.8,u,pg.NewtonConfig(max_iters=5),ex); "
        "print(json.dumps([it.gmres_inner for it in r.iters]))")
out = {}
for v in ("1", "0"):
    env = dict(os.environ, PGMRES_DCGS2=v)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    out["dcgs2" if v == "1" else "cgs2"] = json.loads(r.stdout.strip().splitlines()[-1])
print(json.dumps(out))
