# interleaved A/B of per-step krylov time (scripts/step_breakdown.py) under two environments
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for E in "$ENVA" "$ENVB"; do
    echo "== $E"; env $E timeout 600 python scripts/step_breakdown.py ${PS:-0,2,4} | cut -c1-110
  done
done
