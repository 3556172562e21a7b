#!/bin/bash
# Step-SpMV / whole-solve efficiency vs mesh size (one GPU): bench.py lines
# for n_e in $NES, inputs resident, no e2e / CPU legs.  Output: one JSON line
# per mesh in gpurun_out/size_sweep.jsonl.
NES=${NES:-"31 40 50 62 79 100 125"}
mkdir -p gpurun_out
: > gpurun_out/size_sweep.jsonl
for ne in $NES; do
  python bench.py --ne $ne --steps 3 --warmup 2 --no-e2e --no-cpu-baseline >> gpurun_out/size_sweep.jsonl 2>/dev/null
done
python - <<'PY'
import json
for ln in open("gpurun_out/size_sweep.jsonl"):
    d = json.loads(ln)
    k = d["kernels"]
    print(d["config"]["n_e"], d["config"]["dof"], d["value"], "it/s  step_spmv",
          k["step_spmv"]["GBps"], "update", k["dcgs2_update"]["GBps"],
          "solve_frac", d["solve_roofline"]["frac"], "spmv_frac", d["roofline"]["frac"])
PY
