cd $GRAFT_REPO_ROOT
O=gpurun_out/launch; mkdir -p $O
for P in ${PS:-4}; do
timeout 300 python scripts/profile_step.py --p $P --dim 256 > $O/plain_p$P.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_p$P.csv python scripts/profile_step.py --p $P --dim 256 > $O/ncu_launch_p$P.log 2>&1
echo "rc $?"
done
