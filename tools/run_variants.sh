#!/bin/bash
# Bench (kernel breakdown only) every paper_1906_04051_b200/_lib/var/*/libpgmres.so
cd "$(dirname "$0")/.."
for d in paper_1906_04051_b200/_lib/var/*/; do
  name=$(basename $d)
  PGMRES_LIB=$d/libpgmres.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/var_$name.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/var_$name.json'))
k=d['kernels']
g=lambda n: k.get(n, {}).get('ms_total', 0.0)
print('%-10s %8.1f it/s %7.2f ms  spmv %6.2f  B %6.2f  C/update %6.2f' % ('$name', d['value'], d['ms_per_step'], g('step_spmv'), g('cgs2_passB_update_dots'), g('cgs2_passC_update') + g('dcgs2_update')))"
done
