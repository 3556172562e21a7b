#!/bin/bash
# ncu --set full captures of profile_round.sh only
cd "$(dirname "$0")/.."
# k = 25 of the first cycle: 26th launch of each kernel class
# (-k matches the base function name; the residual SpMV is launch 0 of k_spmv)
ncu --set full --clock-control none --import-source on -k regex:^k_spmv$ -s 26 -c 1 \
    -f -o gpurun_out/ncu_step_spmv python tools/profile_solve.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_cgs2$ -s 25 -c 1 \
    -f -o gpurun_out/ncu_cgs2_b python tools/profile_solve.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_cgs2_update$ -s 25 -c 1 \
    -f -o gpurun_out/ncu_cgs2_c python tools/profile_solve.py > /dev/null 2>&1
for r in step_spmv cgs2_b cgs2_c; do
  python tools/ncu_summary.py gpurun_out/ncu_$r.ncu-rep > gpurun_out/ncu_$r.txt 2>&1
  mv gpurun_out/ncu_$r.ncu-rep /tmp/ 2>/dev/null
done
