#!/bin/bash
# Round-2 evidence refresh, one GPU call (copy gpurun_out/r2_* to profiles/):
#   r2_bench_cfg3.json / _cfg2.json / _ne62.json   python bench.py [--ne ..]
#   r2_bench_ref_cfg3.json / _cfg2.json            python bench.py --impl reference [...]
#   r2_launches_ne{125,50}.txt/.json               ncu launch list (time + DRAM bytes) of one solve
#   r2_ncu_*.txt                                   ncu --set full: step SpMV at k = 25 of cycle 0
#                                                  (r = 0) and of cycle 21 (r = 20), DCGS2 update
set -x
cd "$(dirname "$0")/.."
O=gpurun_out
python bench.py > $O/r2_bench_cfg3.json 2> $O/r2_bench_cfg3.err
python bench.py --ne 50 > $O/r2_bench_cfg2.json 2> $O/r2_bench_cfg2.err
python bench.py --ne 62 --no-cpu-baseline > $O/r2_bench_ne62.json 2> $O/r2_bench_ne62.err
python bench.py --impl reference > $O/r2_bench_ref_cfg3.json 2> $O/r2_bench_ref_cfg3.err
python bench.py --impl reference --ne 50 > $O/r2_bench_ref_cfg2.json 2> $O/r2_bench_ref_cfg2.err
for ne in 125 50; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file /tmp/launches_ne$ne.csv \
      python tools/profile_solve.py --ne $ne > /dev/null 2>&1
  python tools/ncu_launch_summary.py /tmp/launches_ne$ne.csv $O/r2_launches_ne$ne.json \
      > $O/r2_launches_ne$ne.txt
done
# k_spmv launches of a cfg3 solve: 0 = initial residual, then per cycle c the
# m = 50 step SpMVs, the push SpMV and the residual: step k of cycle c is
# launch 1 + 52 c + k (rank during cycle c = min(c, 20))
ncu --set full --clock-control none --import-source on -k regex:^k_spmv$ -s 26 -c 1 \
    -f -o /tmp/r2_ncu_step_spmv_r0 python tools/profile_solve.py --ne 125 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_spmv$ -s 1118 -c 1 \
    -f -o /tmp/r2_ncu_step_spmv_r20 python tools/profile_solve.py --ne 125 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:^k_dcgs2_update$ -s 1075 -c 1 \
    -f -o /tmp/r2_ncu_dcgs2_update_r20 python tools/profile_solve.py --ne 125 > /dev/null 2>&1
for r in step_spmv_r0 step_spmv_r20 dcgs2_update_r20; do
  python tools/ncu_summary.py /tmp/r2_ncu_$r.ncu-rep > $O/r2_ncu_$r.txt 2>&1
done
ls -la $O
