cd $GRAFT_REPO_ROOT
O=gpurun_out
PGMRES_LIB=paper_1906_04051_b200/_lib/var/u4/libpgmres.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O/c13_gputest_u4.log 2>&1; echo "EXIT $?" >> $O/c13_gputest_u4.log
bash tools/ab_interleaved.sh 2 --ne 50 > $O/c13_ab50.txt 2>&1
bash tools/ab_interleaved.sh 2 --ne 62 > $O/c13_ab62.txt 2>&1
bash tools/ab_interleaved.sh 2 > $O/c13_ab125.txt 2>&1
