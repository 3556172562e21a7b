#!/bin/bash
# Run the bench (kernel breakdown only) against every tools/variants/*/libpgmres.so
cd "$(dirname "$0")/.."
for d in tools/variants/*/; do
  name=$(basename $d)
  PGMRES_LIB=$d/libpgmres.so timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/var_$name.json 2>/dev/null
  python -c "
import json,sys
d=json.load(open('gpurun_out/var_$name.json'))
k=d['kernels']
print('$name', d['value'], d['ms_per_step'], 'spmv', k['step_spmv']['GBps'], 'B', k['cgs2_pass2_dots']['GBps'], 'C', k['cgs2_update_norm']['GBps'], 'res', k['residual_spmv']['GBps'])"
done
