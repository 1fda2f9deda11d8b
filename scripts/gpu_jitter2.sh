cd $GRAFT_REPO_ROOT
O=gpurun_out/jit2; mkdir -p $O
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks_throttle_reasons.active,power.draw --format=csv -lms 200 > $O/smi.csv 2>&1 &
SMI=$!
for r in 1 2 3 4 5 6 7 8; do
  echo "run $r $(date +%T.%N)" >> $O/runs.txt
  LDG_TRACE_ITER=1 timeout 120 python scripts/step_breakdown.py 2,4 >> $O/runs.txt 2>&1
done
kill $SMI
grep -v "ldg trace" $O/runs.txt | sed 's/ = assemble.*krylov/ krylov/; s/+ finish.*vcycle/ vcycle/; s/schur.*//'
awk -F, 'NR>1{print $2, $3}' $O/smi.csv | sort | uniq -c | sort -rn | head
