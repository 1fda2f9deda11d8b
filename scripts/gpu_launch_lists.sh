# ncu launch lists (gpu__time_duration, --clock-control none) of one
# implicit-Euler step at 256^2 for each p in $PS.
cd $GRAFT_REPO_ROOT
O=gpurun_out/ll
mkdir -p $O
for P in ${PS:-4 3 2}; do
  timeout 600 python scripts/profile_step.py --p $P --dim 256 > $O/plain_p$P.log 2>&1 && \
  timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_p$P.csv python scripts/profile_step.py --p $P --dim 256 > $O/ncu_p$P.log 2>&1
  echo "p$P rc $?"
done
