# A/B of environment switches on step time (ENVS: ';'-separated env sets, PS degrees)
cd $GRAFT_REPO_ROOT
O=gpurun_out/envs; mkdir -p $O
IFS=';' read -ra LIST <<< "$ENVS"
for r in 1 2; do for E in "${LIST[@]}"; do
  env $E timeout 300 python scripts/step_breakdown.py ${PS:-2,3,4} 2>&1 | sed "s/^/[$E] /"
done; done > $O/ab.txt
cat $O/ab.txt
