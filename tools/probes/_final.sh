cd $GRAFT_REPO_ROOT
O=gpurun_out
python -m pytest tests -m gpu -q > $O/final_gputest.log 2>&1; echo "EXIT $?" >> $O/final_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1
bash tools/profile_round2.sh > $O/final_profile.log 2>&1
