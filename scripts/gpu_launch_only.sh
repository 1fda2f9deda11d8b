# ncu launch lists of one steady-state step per degree (5 warm-up steps)
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-r02_ll}
mkdir -p $O
for P in ${PS:-4 3}; do
  timeout 600 python scripts/profile_step.py --p $P --dim 256 --warmup 5 > $O/plain_p$P.log 2>&1 && \
  timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_p$P.csv python scripts/profile_step.py --p $P --dim 256 --warmup 5 > $O/ncu_launch_p$P.log 2>&1
  echo "launch p$P rc $?" >> $O/rc.txt
done
cat $O/rc.txt
