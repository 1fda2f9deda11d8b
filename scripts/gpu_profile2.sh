cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for P in ${PS:-4 2}; do
timeout 600 python scripts/profile_step.py --p $P --dim 256 > gpurun_out/plain_p$P.log 2>&1 && \
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_p$P.csv python scripts/profile_step.py --p $P --dim 256 > gpurun_out/ncu_p$P.log 2>&1
python scripts/ncu_summary.py gpurun_out/launches_p$P.csv > gpurun_out/launches_p${P}_summary.txt 2>&1
head -22 gpurun_out/launches_p${P}_summary.txt
tail -1 gpurun_out/plain_p$P.log
done
