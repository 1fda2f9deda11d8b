# launch lists (ncu) of one profiled p=$P step under two environments
cd $GRAFT_REPO_ROOT
P=${P:-4}
for E in "$ENVA" "$ENVB"; do
  env $E timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ab_launch.csv python scripts/profile_step.py --p $P --dim 256 > gpurun_out/ab_ncu.log 2>&1
  echo "== $E"; python scripts/ncu_summary.py gpurun_out/ab_launch.csv 2>&1 | head -${NTOP:-16}
  tail -1 gpurun_out/ab_ncu.log
done
