#!/bin/bash
# Interleaved A/B of the libpgmres variants in paper_1906_04051_b200/_lib/var/*:
#   tools/ab_interleaved.sh REPS [bench args]   -> one line per (rep, variant)
cd "$(dirname "$0")/.."
reps=$1; shift
for rep in $(seq 1 $reps); do
  for d in paper_1906_04051_b200/_lib/var/*/; do
    name=$(basename $d)
    PGMRES_LIB=$d/libpgmres.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" > /tmp/ab_$name.json 2>/dev/null
    python -c "
import json
d=json.load(open('/tmp/ab_$name.json'))
k=d['kernels']
g=lambda n: k.get(n, {}).get('ms_total', 0.0)
print('%d %-10s %8.1f it/s %8.2f ms  spmv %7.2f  update %7.2f  ritz %6.2f' % ($rep, '$name', d['value'], d['ms_per_step'], g('step_spmv'), g('dcgs2_update'), g('ritz')))"
  done
done
