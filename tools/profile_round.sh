#!/bin/bash
# One GPU call that refreshes every number under profiles/ (copy the outputs
# from gpurun_out/ after it returns):
#   bench_cfg3.json / bench_cfg2.json   python bench.py (default = cfg3) / --ne 50
#   bench_ref_cfg3.json / _cfg2.json    python bench.py --impl reference [...]
#   launches_ne{125,50}.txt/.json       ncu launch list (time + DRAM bytes) of one solve
#   ncu_*.txt                           ncu --set full of the step SpMV and the DCGS2 update at k = 25 (cfg3)
set -x
cd "$(dirname "$0")/.."
python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --ne 50 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --impl reference > gpurun_out/bench_ref_cfg3.json 2> gpurun_out/bench_ref_cfg3.err
python bench.py --impl reference --ne 50 > gpurun_out/bench_ref_cfg2.json 2> gpurun_out/bench_ref_cfg2.err
for ne in 125 50; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file /tmp/launches_ne$ne.csv \
      python tools/profile_solve.py --ne $ne > /dev/null 2>&1
  python tools/ncu_launch_summary.py /tmp/launches_ne$ne.csv gpurun_out/launches_ne$ne.json \
      > gpurun_out/launches_ne$ne.txt
done
# k = 25 of the first cycle (-k matches the base function name; the residual
# SpMV is launch 0 of k_spmv)
ncu --set full --clock-control none --import-source on -k regex:^k_spmv$ -s 26 -c 1 \
    -f -o /tmp/ncu_step_spmv python tools/profile_solve.py --ne 125 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_dcgs2_update$ -s 25 -c 1 \
    -f -o /tmp/ncu_dcgs2_update python tools/profile_solve.py --ne 125 > /dev/null 2>&1
for r in step_spmv dcgs2_update; do
  python tools/ncu_summary.py /tmp/ncu_$r.ncu-rep > gpurun_out/ncu_$r.txt 2>&1
done
