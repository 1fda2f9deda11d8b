# interleaved medians of step time under several environments (ENVS ';'-separated), ROUNDS rounds
cd $GRAFT_REPO_ROOT
IFS=';' read -ra LIST <<< "$ENVS"
for r in $(seq ${ROUNDS:-2}); do
  for E in "${LIST[@]}"; do
    env $E timeout 600 python scripts/step_breakdown.py ${PS:-0,2,4} | awk -v e="$E" '{print e" | "$1" "$3" "$4" it="$14}' | sed 's/(//'
  done
done
