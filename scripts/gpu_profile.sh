# Launch list of one profiled implicit-Euler step (ncu, gpu__time_duration only).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${P:-4}
DIM=${DIM:-256}
timeout 600 python scripts/profile_step.py --p $P --dim $DIM > gpurun_out/plain_p$P.log 2>&1 && \
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_p$P.csv python scripts/profile_step.py --p $P --dim $DIM > gpurun_out/ncu_p$P.log 2>&1
echo "rc $?"
python scripts/ncu_summary.py gpurun_out/launches_p$P.csv > gpurun_out/launches_p${P}_summary.txt 2>&1
head -30 gpurun_out/launches_p${P}_summary.txt
tail -3 gpurun_out/plain_p$P.log
