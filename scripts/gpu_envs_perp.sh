# per-degree sweep of V-cycle sweep counts (one degree per env set: "P|ENV")
cd $GRAFT_REPO_ROOT
O=gpurun_out/envp; mkdir -p $O
IFS=';' read -ra LIST <<< "$ENVS"
for E in "${LIST[@]}"; do
  P=${E%%|*}; V=${E#*|}
  env $V timeout 300 python scripts/step_breakdown.py $P 2>&1 | sed "s/^/[$V] /"
done > $O/ab.txt
cat $O/ab.txt
