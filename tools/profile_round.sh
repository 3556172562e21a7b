#!/bin/bash
# One GPU call that refreshes every number under profiles/ (copy the outputs
# from gpurun_out/ after it returns):
#   bench_full.json      python bench.py (defaults: cfg2, value + e2e + roofline + cpu baseline)
#   bench_ref.json       python bench.py --impl reference
#   launches.csv/.txt    ncu launch list (time + DRAM bytes) of one cfg2 solve
#   ncu_*.ncu-rep / .txt ncu --set full of the step SpMV, pass B and pass C at k = 25
set -x
cd "$(dirname "$0")/.."
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/profile_solve.py > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt
mv gpurun_out/launches.csv /tmp/
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
